"""Is the DAG replay bound by a per-graph launch rate or a device-wide one? K independent C2 execs
(own chains, own buffers) replayed concurrently on K streams: aggregate replays/s vs one exec."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

dev = torch.device("cuda:0")
spec = wl.c2_chain()
sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(4)]
ptrs = [cgx.ptr_array([t[s.name].data_ptr() for s in spec.externals()]) for t in sets]
n_ext = len(spec.externals())
L = cgx.LIB
for K in (1, 2, 4):
    chains = [runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev)) for _ in range(K)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(K)]
    exs = [chains[k].exec("INDIRECT", stream=streams[k], transport="ROOT_PARAMS") for k in range(K)]
    n = 500
    for i in range(20):
        for k in range(K):
            L.cgx_bind(exs[k].handle, ptrs[(i + k) % 4], n_ext)
            L.cgx_launch(exs[k].handle)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(streams[0])
        for s in streams[1:]:
            s.wait_event(e0)
        for i in range(n):
            for k in range(K):
                L.cgx_bind(exs[k].handle, ptrs[(i + k) % 4], n_ext)
                L.cgx_launch(exs[k].handle)
        for s in streams[1:]:
            ev = torch.cuda.Event()
            ev.record(s)
            streams[0].wait_event(ev)
        e1.record(streams[0])
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    print(json.dumps({"concurrent_execs": K, "us_per_replay_each": best / n,
                      "aggregate_replays_per_s": K * n / (best * 1e-6)}), flush=True)
    for c in chains:
        c.close()
