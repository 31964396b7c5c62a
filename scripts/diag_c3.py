"""Where does the C3 decoder replay time go? CUPTI per-kernel durations (torch.profiler) and
device-timeline replay µs, with and without PDL."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 128
L = int(sys.argv[2]) if len(sys.argv) > 2 else 12
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
spec = wl.c3_chain(T=T, n_layers=L)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
x = runner.host_to_device(wl.slot_values(spec, "x", 0), "bf16", dev)
arr = cgx.ptr_array([x.data_ptr()])
LIB = cgx.LIB
res = {}
for name, mode, xp, nopdl in (("indirect_pdl", "INDIRECT", "FIRST_NODE", False),
                              ("copy_pdl", "COPY", "DEFAULT", False),
                              ("copy_nopdl", "COPY", "DEFAULT", True),
                              ("eager_nopdl", "EAGER", "DEFAULT", True)):
    ex = chain.exec(mode, stream=stream, transport=xp, no_pdl=nopdl)
    for _ in range(3):
        LIB.cgx_bind(ex.handle, arr, 1)
        LIB.cgx_launch(ex.handle)
    stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record(stream)
    for _ in range(n):
        LIB.cgx_bind(ex.handle, arr, 1)
        LIB.cgx_launch(ex.handle)
    e1.record(stream)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    with profile(activities=[ProfilerActivity.CUDA]) as p:
        for _ in range(5):
            LIB.cgx_bind(ex.handle, arr, 1)
            LIB.cgx_launch(ex.handle)
        stream.synchronize()
    per = {}
    for ev in p.key_averages():
        t = getattr(ev, "device_time_total", None)
        if t is None:
            t = getattr(ev, "cuda_time_total", 0.0)
        if t > 0:
            per[ev.key[:70]] = {"count_per_replay": ev.count / 5, "us_per_replay": t / 5,
                                "us_per_launch": t / max(1, ev.count)}
    res[name] = {"replay_us": us, "kernels": per}
    ex.close()
print(json.dumps(res, indent=1))
chain.close()
