"""C4 — input-size sweep exercising the graph-vs-eager cost-benefit selector.

For S = 1 KiB .. 1 GiB per input (3 inputs), window mode (kernels touch 4096 elements, so the
COPY arm's copy dominates) and full mode (kernels read all of S), profile the three candidate
modules with cgx_profile_ex (slow path; 2 rotating input sets, each arm's rebinding
delta against its own launch-only loop, the dependency-DAG estimate model) and decide with
cgx_select twice: with {EAGER, COPY, INDIRECT} and with PI disabled (the PyTorch2-style world).
The decisions are re-derived by the CPU oracle (oracle/selector.py) from the same numbers and must
match exactly, in both decision modes (measured totals / estimates). Each point also reports the
estimate error of every arm against its measured total.

The whole sweep runs `--sweeps` times (default 3); the crossover S* where the PI-less selector
flips to EAGER is reported per sweep and as their median (one sweep is not a result).
Usage: c4_sweep.py [window] [full] [--sweeps N]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from oracle import selector as osel  # noqa: E402
from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import splitmix as sm  # noqa: E402
from synth import workloads as wl  # noqa: E402


def one_point(mode, S, dev, sh, n_sets=2):
    spec = wl.c4_chain(S, window_mode=(mode == "window"))
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    sets = []
    for r in range(n_sets):
        ins = []
        for s in spec.externals():
            t = torch.empty(s.nelems, dtype=torch.float32, device=dev)
            cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED, sm.stream_id(spec.index(s.name), r), sh)
            ins.append(t)
        sets.append(ins)
    torch.cuda.synchronize()
    reps = 200 if S <= (16 << 20) else 20
    p = cgx.profile(chain.handle, -1, None, reps, sh, sets=[[t.data_ptr() for t in ins] for ins in sets])
    d = p.as_dict()
    prof = p.oracle_dict()
    dec, _ = cgx.select([p])
    p.ind_available = 0
    dec_nopi, _ = cgx.select([p])
    o_dec = osel.select([dict(prof, ind_available=True)])[0]
    o_nopi = osel.select([dict(prof, ind_available=False)])[0]
    p.ind_available, p.use_measured = 1, 0
    dec_est, est_est = cgx.select([p])
    o_est = osel.estimates(dict(prof, use_measured=False))
    err = {k: (e - m) / m for k, e, m in zip(("eager", "copy", "ind"), est_est[0],
                                             (d["t_eager_us"], d["t_copy_us"], d["t_ind_us"]))}
    pt = {"mode": mode, "S_bytes": S, "t_eager_us": d["t_eager_us"], "t_copy_us": d["t_copy_us"],
          "t_ind_us": d["t_ind_us"], "c_copy_us": d["c_copy_us"], "c_ind_us": d["c_ind_us"],
          "t_copy_base_us": d["t_copy_base_us"], "t_ind_base_us": d["t_ind_base_us"],
          "L_us": d["L_us"], "G_us": d["G_us"], "delta_us": d["delta_us"], "lambda_us": d["lambda_us"],
          "span_us": d["span_us"], "est_us": list(est_est[0]), "est_rel_err": err,
          "ind_transport": cgx.XPORT_NAME.get(d["ind_transport"], d["ind_transport"]),
          "decision": cgx.DECIDE[dec[0]], "decision_no_pi": cgx.DECIDE[dec_nopi[0]],
          "decision_estimates": cgx.DECIDE[dec_est[0]],
          "oracle_agrees": (o_dec == dec[0] and o_nopi == dec_nopi[0] and tuple(est_est[0]) == tuple(o_est) and
                            osel.select([dict(prof, use_measured=False)])[0] == dec_est[0]),
          "graph_not_slower_than_eager_full": d["t_ind_us"] <= d["t_eager_us"]}
    chain.close()
    del sets
    torch.cuda.empty_cache()
    return pt


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    n_sweeps = int(sys.argv[sys.argv.index("--sweeps") + 1]) if "--sweeps" in sys.argv else 3
    args = [a for a in args if not a.isdigit()]
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    out = {"points": [], "sweeps": n_sweeps}
    modes = args or ["window", "full"]
    for sweep in range(n_sweeps):
        for mode in modes:
            for S in wl.C4_SIZES:
                if mode == "full" and S > (256 << 20):
                    continue
                pt = one_point(mode, S, dev, sh)
                pt["sweep"] = sweep
                out["points"].append(pt)
                print(json.dumps(pt), flush=True)
    for mode in modes:
        xs = []
        for sweep in range(n_sweeps):
            pts = [p for p in out["points"] if p["mode"] == mode and p["sweep"] == sweep]
            flip = [p["S_bytes"] for p in pts if p["decision_no_pi"] == "EAGER"]
            xs.append(min(flip) if flip else None)
        out[f"crossover_no_pi_{mode}_per_sweep"] = xs
        # monotone crossover: the smallest S from which the PI-less selector keeps choosing EAGER at
        # every larger size (below it, eager and graph+copy are within noise of each other)
        mono = []
        for sweep in range(n_sweeps):
            pts = sorted((p for p in out["points"] if p["mode"] == mode and p["sweep"] == sweep), key=lambda p: p["S_bytes"])
            m = None
            for p in reversed(pts):
                if p["decision_no_pi"] != "EAGER":
                    break
                m = p["S_bytes"]
            mono.append(m)
        out[f"crossover_monotone_no_pi_{mode}_per_sweep"] = mono
        vals = [x for x in xs if x is not None]
        out[f"crossover_no_pi_{mode}_median"] = statistics.median(vals) if len(vals) == len(xs) and vals else None
        pts = [p for p in out["points"] if p["mode"] == mode]
        out[f"all_oracle_agree_{mode}"] = all(p["oracle_agrees"] for p in pts)
        errs = [abs(v) for p in pts for v in p["est_rel_err"].values()]
        out[f"est_rel_err_{mode}"] = {"median": statistics.median(errs), "max": max(errs)}
        if mode == "full":
            out["full_graph_not_slower_than_eager"] = all(p["graph_not_slower_than_eager_full"] for p in pts)
    print(json.dumps({k: v for k, v in out.items() if k != "points"}))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c4_sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
