"""Where does the C2 replay time go? The deployed replay (INDIRECT / FIRST_NODE, dataflow sync)
timed with the real kernels reduced step by step (runtime debug knobs, one subprocess each):

  full                 the deployed replay
  CGX_DEBUG_NOOP=2     synchronisation kept (dataflow waits + signals), memory work skipped
  CGX_DEBUG_NOOP=1     every kernel returns right after its PDL trigger: the pure launch cascade
                       of the real kernels (grids, block sizes, parameter blocks)
plus grid caps (CGX_CHAIN_MAX_CTAS) for each.
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
    spec = wl.c2_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(4)]
    stream = torch.cuda.current_stream()
    ex = chain.exec("INDIRECT", stream=stream, transport=os.environ.get("XPORT", "FIRST_NODE"), sync=sys.argv[2],
                    graph_streams=int(sys.argv[3]) if len(sys.argv) > 3 else 0)
    ptrs = [cgx.ptr_array([t[s.name].data_ptr() for s in spec.externals()]) for t in sets]
    n_ext = len(spec.externals())
    L = cgx.LIB
    for i in range(50):
        L.cgx_bind(ex.handle, ptrs[i % 4], n_ext)
        L.cgx_launch(ex.handle)
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for i in range(500):
            L.cgx_bind(ex.handle, ptrs[i % 4], n_ext)
            L.cgx_launch(ex.handle)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 500)
    print(json.dumps({"us_per_replay": best}))
    ex.close()
    chain.close()
    sys.exit(0)


def run(env_extra, sync="AUTO", streams=0):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, __file__, "child", sync, str(streams)], env=env, capture_output=True,
                       text=True, timeout=240)
    try:
        return json.loads(r.stdout.strip().splitlines()[-1])["us_per_replay"]
    except (IndexError, ValueError, KeyError):
        return r.stderr[-400:]


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "graph":
    # dependency-DAG capture (sync GRAPH): capture streams x grid cap x transport
    for xp in ("FIRST_NODE", "H2D", "ROOT_PARAMS"):
        for streams in (2, 4, 8, 16, 32):
            for cap in (None, "148"):
                e = {"XPORT": xp}
                if cap:
                    e["CGX_CHAIN_MAX_CTAS"] = cap
                key = f"sync=GRAPH xport={xp} streams={streams} cap={cap or 'default'}"
                print(json.dumps({key: run(e, "GRAPH", streams)}), flush=True)
    print(json.dumps({"sync=AUTO xport=FIRST_NODE": run({}, "AUTO")}), flush=True)
    print(json.dumps({"sync=CHAIN xport=FIRST_NODE": run({}, "CHAIN")}), flush=True)
elif __name__ == "__main__":
    out = {}
    for sync in ("AUTO",):
        for cap in (None, "16", "4"):
            for mode in (None, "2", "1"):
                e = {}
                if cap:
                    e["CGX_CHAIN_MAX_CTAS"] = cap
                if mode:
                    e["CGX_DEBUG_NOOP"] = mode
                key = f"sync={sync} cap={cap or 'default'} noop={mode or 'off'}"
                out[key] = run(e, sync)
                print(json.dumps({key: out[key]}), flush=True)
