"""C3 decode shapes (T = 1, 2, 4, 8): 12-layer replay µs with the small-M GEMV path vs the tcgen05
kernel forced (CGX_GEMM_NO_GEMV=1), INDIRECT / FIRST_NODE."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.current_stream()
for T in (1, 2, 4, 8):
    for nogemv in ("0", "1"):
        os.environ["CGX_GEMM_NO_GEMV"] = nogemv
        spec = wl.c3_chain(T=T, n_layers=12)
        chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
        xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
        ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
        ex = chain.exec("INDIRECT", stream=stream, transport="FIRST_NODE")
        for i in range(20):
            cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            cgx.LIB.cgx_launch(ex.handle)
        best = 1e9
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
        print(json.dumps({"T": T, "gemm": "gemv" if nogemv == "0" else "tcgen05", "us_per_replay": best}), flush=True)
        chain.close()
