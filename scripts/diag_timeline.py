"""Diagnostic: per-node timeline of one C2 replay (CGX_NODE_TRACE=1) for each sync mode.
Prints, per launch position, entry / ready / exit in µs relative to the first entry."""
import json
import os
import sys

os.environ["CGX_NODE_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
spec = wl.c2_chain()
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(2)]
res = {}
for sync in sys.argv[1:] or ["AUTO", "CHAIN"]:
    ex = chain.exec("INDIRECT", transport="FIRST_NODE", sync=sync)
    for i in range(20):
        ex.bind(sets[i % 2])
        ex.launch()
    K = len(spec.nodes)
    rows = []
    for rep in range(3):
        cgx.node_trace(ex.handle, K)            # sync + reset
        ex.bind(sets[rep % 2])
        ex.launch()
        tr = cgx.node_trace(ex.handle, K)
        t0 = min(t[0] for t in tr)
        rows = [((a - t0) / 1e3, (b - t0) / 1e3, (c - t0) / 1e3) for a, b, c in tr]
    res[sync] = rows
    span = max(r[2] for r in rows)
    print(f"== {sync}: span {span:.1f} us")
    for p, (a, b, c) in enumerate(rows):
        n = spec.nodes[p]
        print(f"{p:3d} {n.op:10s} {spec.slot(n.out).nelems:8d}  entry {a:7.2f}  ready {b:7.2f}  exit {c:7.2f}  dur {c - a:6.2f}")
    ex.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/diag_timeline.json", "w"))
