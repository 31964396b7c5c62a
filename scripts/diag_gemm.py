"""Per-CTA phase timeline of the decoder GEMM nodes (cgx_debug_gemm_trace): where do the µs go?"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_19779_b200 import build
build.build()
from paper_2503_19779_b200 import cgx, runner
from synth import workloads as wl
dev = torch.device("cuda:0")
spec = wl.c3_chain(T=128, n_layers=1)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
ex = chain.exec("COPY")
x = runner.host_to_device(wl.slot_values(spec, "x", 0), "bf16", dev)
ex.bind({"x": x}); ex.launch(); torch.cuda.synchronize()
names = ["entry", "setup", "stage0", "mma_issued", "stored", "pushed", "arrived", "exit", "acc_ready", "acc_regs", "staged"]
for pos, node in enumerate(spec.nodes):
    if node.op != "GEMM_BF16":
        continue
    for rep in range(3):
        tr = np.array(cgx.gemm_trace(ex.handle, pos), dtype=np.float64)
    t0 = tr[:, 0].min()
    rel = (tr - t0) / 1e3          # us relative to the first CTA entry
    rel[tr == 0] = np.nan
    a = node.attrs
    print(f"GEMM {a['M']}x{a['N']}x{a['K']} ctas={len(tr)}")
    for i, nm in enumerate(names):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"   {nm:10s} min {np.nanmin(col):7.2f}  med {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")
chain.close()
