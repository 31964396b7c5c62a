"""Per-CTA phase timeline of the decoder GEMM nodes (cgx_debug_gemm_trace): where do the µs go?

Default: %globaltimer stamps relative to the first CTA entry (256 ns tick). --clk: SM clock64
stamps (CGX_GEMM_TRACE_CLK=1), reported per CTA relative to its own entry in µs at the SM clock
(cycle-exact, only comparable within a CTA). --fused: the fused-residual chain with the LayerNorms
folded into their GEMMs (fuse = CGX_FUSE_LN_GEMM); --attn: and the attention folded into the O-proj
(fuse |= CGX_FUSE_ATTN_GEMM; slots 12 / 13 / 14 = Q-K-V landed / warp 2 / other warps done).
Usage: diag_gemm.py [--clk] [--fused] [--attn]"""
import os
import sys

CLK = "--clk" in sys.argv
if "--attn" in sys.argv:
    os.environ["CGX_ATTN_GEMM_TC"] = "1"
if CLK:
    os.environ["CGX_GEMM_TRACE_CLK"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

fused = "--fused" in sys.argv
SM_GHZ = 1.965
dev = torch.device("cuda:0")
spec = wl.c3_chain(T=128, n_layers=2 if fused else 1, fuse_residual=fused)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
ex = chain.exec("COPY", fuse=(cgx.FUSE_LN_GEMM if fused else 0) | (cgx.FUSE_ATTN_GEMM if "--attn" in sys.argv else 0))
x = runner.host_to_device(wl.slot_values(spec, "x", 0), "bf16", dev)
ex.bind({"x": x})
ex.launch()
torch.cuda.synchronize()
# slot -> phase (k_gemm.cu trace_at): 2 = first A/W group landed (MMA warp), 15 = last UMMA issued,
# 3 = accumulator commit issued, 8 / 9 = accumulator ready / in registers (epilogue), 10 = partial
# staged, 5 = peer pushes issued, 6 = peers' rows arrived, 4 = outputs stored, 11 = A loads issued
names = ["entry", "setup", "stage0", "mma_issued", "stored", "pushed", "arrived", "exit", "acc_ready", "acc_regs",
         "staged", "a_issued", "q0_done", "q1_done", "q2_done", "mma_loop"]
lnodes = cgx.launch_nodes(ex.handle)
for pos, k in enumerate(lnodes):
    node = spec.nodes[k]
    if node.op != "GEMM_BF16":
        continue
    for rep in range(3):
        tr = np.array(cgx.gemm_trace(ex.handle, pos), dtype=np.float64)
    if CLK:
        rel = (tr - tr[:, :1]) / (SM_GHZ * 1e3)   # µs from this CTA's own entry
    else:
        rel = (tr - tr[:, 0].min()) / 1e3         # µs from the first CTA entry
    rel[tr == 0] = np.nan
    a = node.attrs
    folded = pos > 0 and spec.nodes[k - 1].op == "LAYERNORM" and (k - 1) not in lnodes
    print(f"GEMM {a['M']}x{a['N']}x{a['K']}{' +LN' if folded else ''} ctas={len(tr)} "
          f"({'clock64, per CTA' if CLK else 'globaltimer'})")
    for i, nm in enumerate(names):
        col = rel[:, i]
        if not nm or np.all(np.isnan(col)):
            continue
        print(f"   {nm:10s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")
chain.close()
