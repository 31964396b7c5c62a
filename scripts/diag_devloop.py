"""NEXT-4 diagnostic: µs per replay, host-driven (cgx_bind + cgx_launch per replay, H2D and DEVICE
transports) vs device-driven (one cgx_device_loop of N replays), C1 and C2, 8 rotating sets."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import splitmix as sm  # noqa: E402
from synth import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
sh = stream.cuda_stream
LIB = cgx.LIB
res = {}
for cfg in sys.argv[1:] or ["C1", "C2"]:
    spec = wl.c2_chain() if cfg == "C2" else wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ext = spec.externals()
    R = 8
    sets, ptrs = [], []
    for r in range(R):
        ts = [torch.empty(s.nelems, dtype=torch.float32, device=dev) for s in ext]
        for s, t in zip(ext, ts):
            cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED, sm.stream_id(spec.index(s.name), r), sh)
        sets.append(ts)
        ptrs.append(cgx.ptr_array([t.data_ptr() for t in ts]))
    table = torch.tensor([[t.data_ptr() for t in ts] for ts in sets], dtype=torch.int64, device=dev)
    torch.cuda.synchronize()
    N = 2000

    def ev_time(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            fn()
            e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / N

    out = {}
    for xp in ("H2D", "DEVICE"):
        ex = chain.exec("INDIRECT", stream=stream, transport=xp)

        def host_loop():
            for i in range(N):
                LIB.cgx_bind(ex.handle, ptrs[i % R], len(ext))
                LIB.cgx_launch(ex.handle)
        host_loop()
        out[f"host_loop_{xp}"] = min(ev_time(host_loop) for _ in range(3))
        stream.synchronize()
        t0 = time.process_time()
        host_loop()
        out[f"host_loop_{xp}_cpu_us"] = (time.process_time() - t0) * 1e6 / N
        stream.synchronize()
        if xp == "DEVICE":
            def dev_loop():
                cgx.device_loop(ex.handle, table.data_ptr(), R, N)
            dev_loop()
            out["device_loop"] = min(ev_time(dev_loop) for _ in range(3))
            stream.synchronize()
            t0 = time.process_time()
            dev_loop()
            out["device_loop_cpu_us"] = (time.process_time() - t0) * 1e6 / N
            stream.synchronize()
        ex.close()
    res[cfg] = out
    print(cfg, json.dumps(out), flush=True)
    chain.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/diag_devloop.json", "w"), indent=1)
