"""DAG capture issue order (runtime.cu capture_dag, CGX_DAG_ORDER): chain order vs longest-path-first
list scheduling, on the deployed replays (sync AUTO). One subprocess per (workload, order), the two
orders interleaved over several rounds so box drift shows up as spread, not as a difference.

    python scripts/diag_dag_order.py            # prints one JSON line per measurement + a summary
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2503_19779_b200 import cgx, runner
    from synth import workloads as wl
    dev = torch.device("cuda:0")
    work, mode, xp = sys.argv[2], sys.argv[3], sys.argv[4]
    stream = torch.cuda.Stream()
    L = cgx.LIB
    if work == "train":
        spec = wl.mlp_train_chain(n_blocks=6)
    elif work == "c3":
        spec = wl.c3_chain(T=128, n_layers=12)
    else:
        spec = wl.c2_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(4)]
    ptrs = [cgx.ptr_array([t[n].data_ptr() for n in chain.ext_names]) for t in sets]
    n_ext = len(chain.ext_names)
    kw = {}
    if work == "train":
        f0, l0 = spec.segments[0]
        f1, l1 = spec.segments[1]
        init = chain.exec("EAGER", stream=stream, first_node=f0, n_nodes=l0 - f0 + 1)
        L.cgx_bind(init.handle, ptrs[0], n_ext)
        L.cgx_launch(init.handle)
        kw = dict(first_node=f1, n_nodes=l1 - f1 + 1)
    ex = chain.exec(mode, stream=stream, transport=xp, sync="AUTO", **kw)
    for i in range(30):
        L.cgx_bind(ex.handle, ptrs[i % 4], n_ext)
        L.cgx_launch(ex.handle)
    n = 300 if work == "c2" else 100
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for i in range(n):
            L.cgx_bind(ex.handle, ptrs[i % 4], n_ext)
            L.cgx_launch(ex.handle)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    print(json.dumps({"us_per_replay": best, "dag_streams": ex.stats()["dag_streams"]}))
    ex.close()
    chain.close()
    sys.exit(0)

CASES = [("c2", "INDIRECT", "FIRST_NODE"), ("c2", "INDIRECT", "H2D"), ("c2", "COPY", "DEFAULT"),
         ("train", "INDIRECT", "ROOT_PARAMS")]


def run(case, order):
    env = dict(os.environ, CGX_DAG_ORDER=order)
    r = subprocess.run([sys.executable, __file__, "child", *case], env=env, capture_output=True, text=True,
                       timeout=300)
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])
    except (IndexError, ValueError):
        return {"error": r.stderr[-300:]}


def main():
    res = {}
    for rnd in range(2):
        for case in CASES:
            for order in ("chain", "priority", "level"):
                out = run(case, order)
                key = "/".join(case) + f" order={order}"
                res.setdefault(key, []).append(out.get("us_per_replay"))
                print(json.dumps({"round": rnd, "case": key, **out}), flush=True)
    summ = {k: min(v for v in vs if v) if any(vs) else None for k, vs in res.items()}
    print(json.dumps({"summary_min_us": summ}))
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump({"runs": res, "min_us": summ}, open(os.path.join(ROOT, "gpurun_out", "dag_order.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
