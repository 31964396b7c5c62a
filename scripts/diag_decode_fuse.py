"""T = 1 decode (12 layers, INDIRECT FIRST_NODE, best of 3 x 300 replays): the unfused and the
fused-residual chains with each capture-time fusion (fuse bits)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
res = {}
for fr in (False, True):
    spec = wl.c3_chain(T=1, n_layers=12, fuse_residual=fr)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
    ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
    for name, fz in (("none", 0), ("add_ln", cgx.FUSE_ADD_LN), ("ln_gemm", cgx.FUSE_LN_GEMM),
                     ("ln_attn_gemm", cgx.FUSE_LN_GEMM | cgx.FUSE_ATTN_GEMM)):
        ex = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", fuse=fz)
        for i in range(20):
            cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            cgx.LIB.cgx_launch(ex.handle)
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(300):
                cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
                cgx.LIB.cgx_launch(ex.handle)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / 300)
        res[f"{'fused_residual' if fr else 'unfused'}/{name}"] = {"us": round(best, 1),
                                                                   "launches": ex.stats()["kernels_per_replay"]}
        ex.close()
    chain.close()
for k, v in res.items():
    print(k, v, f"{12 * 14.16e6 / (v['us'] * 1e-6) / 1e9:.0f} GB/s of weights")
