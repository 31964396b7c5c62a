"""Replay timeline of the C3 decoder (CGX_NODE_TRACE=1): per node, first CTA entry, last CTA past its
PDL wait ("ready") and last CTA exit, in µs from the first entry of the replay (INDIRECT,
ROOT_PARAMS, best of 5 replays by span). Per op class: mean post-wait work (exit - ready) and mean
critical-path gap (ready - predecessor exit: the launch / dependency-resolution latency the chain
pays per node). Usage: diag_c3_timeline.py [T] [layers] [--fuse] [--ln-gemm] [--attn-gemm]"""
import json
import os
import sys

os.environ["CGX_NODE_TRACE"] = "1"
if "--attn-gemm" in sys.argv:
    os.environ["CGX_ATTN_GEMM_TC"] = "1"   # (the tcgen05 attention fold is a measurement knob)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
T = int(args[0]) if args else 128
L = int(args[1]) if len(args) > 1 else 12
fuse = "--fuse" in sys.argv or "--ln-gemm" in sys.argv
ln_gemm = "--ln-gemm" in sys.argv
dev = torch.device("cuda:0")
spec = wl.c3_chain(T=T, n_layers=L, fuse_residual=fuse)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(2)]
fz = (cgx.FUSE_LN_GEMM if ln_gemm else 0) | (cgx.FUSE_ATTN_GEMM if "--attn-gemm" in sys.argv else 0)
ex = chain.exec("INDIRECT", fuse=fz)
for i in range(20):
    ex.bind({"x": xs[i % 2]})
    ex.launch()
lnodes = cgx.launch_nodes(ex.handle)   # chain node per launch position (fusion: fewer launches)
K = len(lnodes)
best = None
for rep in range(5):
    cgx.node_trace(ex.handle, K)
    ex.bind({"x": xs[rep % 2]})
    ex.launch()
    tr = cgx.node_trace(ex.handle, K)
    t0 = min(t[0] for t in tr)
    rows = [((a - t0) / 1e3, (b - t0) / 1e3, (c - t0) / 1e3) for a, b, c in tr]
    span = max(r[2] for r in rows)
    if best is None or span < best[0]:
        best = (span, rows)
span, rows = best
print(f"== C3 T={T} L={L} fuse={fuse}: span {span:.1f} us over {K} nodes ({span / K:.2f} us/node)")
agg = {}
prev_exit = 0.0
for p, (a, b, c) in enumerate(rows):
    n = spec.nodes[lnodes[p]]
    key = n.op if n.op != "GEMM_BF16" else f"GEMM {n.attrs['N']}x{n.attrs['K']}"
    if ln_gemm and n.op == "GEMM_BF16" and lnodes[p] > 0 and spec.nodes[lnodes[p] - 1].op == "LAYERNORM" \
            and (p == 0 or lnodes[p - 1] != lnodes[p] - 1):
        key += " +LN"
    d = agg.setdefault(key, [0, 0.0, 0.0])
    d[0] += 1
    d[1] += c - b
    d[2] += b - prev_exit
    if p < 2 * (K // L) + 2:
        print(f"{p:3d} {key:18s} entry {a:8.2f} ready {b:8.2f} exit {c:8.2f}  work {c - b:6.2f}  gap {b - prev_exit:6.2f}")
    prev_exit = c
print(f"{'op':18s} {'n':>4s} {'work_mean':>10s} {'gap_mean':>9s} {'(work+gap)_sum':>15s}")
for k, (n, work, gap) in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][2])):
    print(f"{k:18s} {n:4d} {work / n:10.2f} {gap / n:9.2f} {work + gap:15.1f}")
os.makedirs("gpurun_out", exist_ok=True)
json.dump({"span": span, "rows": rows, "ops": [n.op for n in spec.nodes]},
          open(f"gpurun_out/c3_timeline_T{T}{'_fuse' if fuse else ''}.json", "w"))
ex.close()
chain.close()
