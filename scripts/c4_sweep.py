"""C4 — input-size sweep exercising the graph-vs-eager cost-benefit selector.

For S = 1 KiB .. 1 GiB per input (3 inputs), window mode (kernels touch 4096 elements, so the
COPY arm's copy dominates) and full mode (kernels read all of S), profile the three candidate
modules with cgx_profile (slow path) and decide with cgx_select twice: with
{EAGER, COPY, INDIRECT} and with PI disabled (the PyTorch2-style world). The decisions are
re-derived by the CPU oracle (oracle/selector.py) from the same numbers and must match exactly.
Reports the crossover S* where the PI-less selector flips to EAGER (the EOS-like regime).
"""
import json
import os
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


def main():
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    out = {"points": []}
    modes = sys.argv[1:] or ["window", "full"]
    for mode in modes:
        for S in wl.C4_SIZES:
            if mode == "full" and S > (256 << 20):
                continue
            spec = wl.c4_chain(S, window_mode=(mode == "window"))
            chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
            ins = []
            for s in spec.externals():
                t = torch.empty(s.nelems, dtype=torch.float32, device=dev)
                cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED, sm.stream_id(spec.index(s.name), 0), sh)
                ins.append(t)
            torch.cuda.synchronize()
            reps = 200 if S <= (16 << 20) else 20
            p = cgx.profile(chain.handle, -1, [t.data_ptr() for t in ins], reps, sh)
            d = p.as_dict()
            dec, est = cgx.select([p])
            p.ind_available = 0
            dec_nopi, _ = cgx.select([p])
            prof = dict(L=d["L_us"], G=d["G_us"], delta=d["delta_us"], d=d["d_us"], c_copy=d["c_copy_us"],
                        c_ind=d["c_ind_us"], F=d["F_us"], use_measured=True, t_eager=d["t_eager_us"],
                        t_copy=d["t_copy_us"], t_ind=d["t_ind_us"])
            o_dec = osel.select([prof])[0]
            o_nopi = osel.select([dict(prof, ind_available=False)])[0]
            prof_est = dict(prof, use_measured=False)
            o_est = osel.estimates(prof_est)
            p.ind_available, p.use_measured = 1, 0
            dec_est, est_est = cgx.select([p])
            pt = {"mode": mode, "S_bytes": S, "t_eager_us": d["t_eager_us"], "t_copy_us": d["t_copy_us"],
                  "t_ind_us": d["t_ind_us"], "c_copy_us": d["c_copy_us"], "c_ind_us": d["c_ind_us"],
                  "L_us": d["L_us"], "G_us": d["G_us"], "delta_us": d["delta_us"],
                  "decision": cgx.DECIDE[dec[0]], "decision_no_pi": cgx.DECIDE[dec_nopi[0]],
                  "decision_estimates": cgx.DECIDE[dec_est[0]],
                  "oracle_agrees": (o_dec == dec[0] and o_nopi == dec_nopi[0] and
                                    tuple(est_est[0]) == tuple(o_est) and
                                    osel.select([prof_est])[0] == dec_est[0])}
            out["points"].append(pt)
            print(json.dumps(pt), flush=True)
            chain.close()
            del ins
            torch.cuda.empty_cache()
    for mode in modes:
        pts = [p for p in out["points"] if p["mode"] == mode]
        flip = [p["S_bytes"] for p in pts if p["decision_no_pi"] == "EAGER"]
        out[f"crossover_no_pi_{mode}"] = min(flip) if flip else None
        out[f"all_oracle_agree_{mode}"] = all(p["oracle_agrees"] for p in pts)
    print(json.dumps({k: v for k, v in out.items() if k != "points"}))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "c4_sweep.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
