"""K-split sweep of the decoder GEMMs (CGX_GEMM_TILING, read at exec build time) on the deployed arm:
C3 12 layers, T = 128, fused residual + LN folded, INDIRECT FIRST_NODE; one shape varied at a time
from the default tiling, 3 rounds interleaved, best of 3 x 200 replays each (us per replay)."""
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
spec = wl.c3_chain(T=128, n_layers=12, fuse_residual=True)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
CANDS = [None, "768x768=32/6", "768x768=32/3", "768x768=32/8", "768x3072=32/6", "768x3072=32/12",
         "768x3072=32/16", "3072x768=32/1", "3072x768=32/3", "2304x768=32/3"]
if len(sys.argv) > 1:
    CANDS = [None] + sys.argv[1:]
execs = {}
for c in CANDS:
    if c:
        os.environ["CGX_GEMM_TILING"] = c
    else:
        os.environ.pop("CGX_GEMM_TILING", None)
    try:
        execs[c] = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE", fuse=cgx.FUSE_LN_GEMM)
    except cgx.CgxError as exn:
        print(json.dumps({"tiling": c, "error": str(exn)}))
os.environ.pop("CGX_GEMM_TILING", None)
res = {c: [] for c in execs}
for rnd in range(3):
    for c, ex in execs.items():
        for i in range(20):
            cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            cgx.LIB.cgx_launch(ex.handle)
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(200):
                cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
                cgx.LIB.cgx_launch(ex.handle)
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / 200)
        res[c].append(round(best, 1))
for c, v in res.items():
    print(json.dumps({"tiling": c or "default", "launches": execs[c].stats()["kernels_per_replay"], "us": v}))
