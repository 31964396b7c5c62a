"""A/B of the attention Q-fragment loads (CGX_ATTN_QALL=1: every warp, the round-1 kernel; 0: only the
warps owning a key chunk, the default) on the C3
chain (12 layers, fused residual + LN folded, INDIRECT FIRST_NODE), alternating 4 times in one
process, best of 3 x 300 replays each."""
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
T = int(sys.argv[1]) if len(sys.argv) > 1 else 128
spec = wl.c3_chain(T=T, n_layers=12, fuse_residual=True)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
execs = {}
for v in ("1", "0"):
    os.environ["CGX_ATTN_QALL"] = v
    execs[v] = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", fuse=cgx.FUSE_LN_GEMM)
res = {"1": [], "0": []}
for rnd in range(4):
    for v, ex in execs.items():
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
        res[v].append(round(best, 1))
print(f"C3 T={T} fused residual + LN folded, us per replay: Q loaded by every warp {res['1']}  by the chunk owners {res['0']}")
