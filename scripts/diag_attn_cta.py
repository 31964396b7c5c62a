"""Per-CTA phases of the C3 attention nodes inside the deployed replay (CGX_CTA_TRACE=1): for each
ATTN launch of the fused-residual, LN-folded 12-layer chain (INDIRECT, T = 128), the distribution
over CTAs of entry / past-wait / K-V staged / partials published / exit, in µs from the FIRST CTA
past its PDL wait of that node. Usage: diag_attn_cta.py [T] [layers]"""
import os
import sys

os.environ["CGX_CTA_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
T = int(args[0]) if args else 128
L = int(args[1]) if len(args) > 1 else 12
dev = torch.device("cuda:0")
spec = wl.c3_chain(T=T, n_layers=L, fuse_residual=True)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(2)]
ex = chain.exec("INDIRECT", fuse=cgx.FUSE_LN_GEMM)
for i in range(30):
    ex.bind({"x": xs[i % 2]})
    ex.launch()
torch.cuda.synchronize()
lnodes = cgx.launch_nodes(ex.handle)
pos = [p for p, n in enumerate(lnodes) if spec.nodes[n].op == "ATTN_CAUSAL"]
names = ["entry", "waited", "kv_staged", "published", "exit"]
agg = {k: [] for k in names}
per_qb = {}
for p in pos[1:]:   # (layer 0's attention follows the first GEMM)
    tr = np.array(cgx.cta_trace(ex.handle, p), dtype=np.float64)[:, :5]
    t0 = tr[:, 1].min()
    rel = (tr - t0) / 1e3
    rel[tr == 0] = np.nan
    for i, k in enumerate(names):
        agg[k].append(rel[:, i])
    gx = (T + 15) // 16
    for c in range(tr.shape[0]):
        per_qb.setdefault(c % gx, []).append(rel[c, 4] - rel[c, 1])
print(f"== C3 T={T} L={L} attention CTAs (fused residual, LN folded, INDIRECT), µs from the first CTA past its wait")
for k in names:
    v = np.concatenate(agg[k])
    v = v[~np.isnan(v)]
    if v.size:
        print(f"  {k:10s} min {v.min():6.2f}  p10 {np.percentile(v, 10):6.2f}  med {np.median(v):6.2f}  "
              f"p90 {np.percentile(v, 90):6.2f}  max {v.max():6.2f}")
print("  per query block: median (exit - waited) µs")
for qb in sorted(per_qb):
    print(f"    qblock {qb}: {np.nanmedian(per_qb[qb]):.2f}")
