"""Diagnostic: C2 (and C1) replay time per node-synchronisation mode.
Device-timeline µs per bind+launch over N back-to-back replays, 8 rotating input sets."""
import json
import os
import sys

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
for cfg in sys.argv[1:] or ["C2", "C1"]:
    spec = wl.c2_chain() if cfg == "C2" else wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ext = spec.externals()
    R = 8
    sets = []
    for r in range(R):
        ts = [torch.empty(s.nelems, dtype=torch.float32, device=dev) for s in ext]
        for s, t in zip(ext, ts):
            cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED, sm.stream_id(spec.index(s.name), r), sh)
        sets.append((ts, cgx.ptr_array([t.data_ptr() for t in ts])))
    torch.cuda.synchronize()

    def timed(h, n):
        for i in range(20):
            LIB.cgx_bind(h, sets[i % R][1], len(ext))
            LIB.cgx_launch(h)
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(n):
                assert LIB.cgx_bind(h, sets[i % R][1], len(ext)) == 0, cgx.last_error()
                assert LIB.cgx_launch(h) == 0, cgx.last_error()
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        return best
    out = {}
    for name, mode, xp, kw in [("ind_t5_auto", "INDIRECT", "FIRST_NODE", {}),
                               ("ind_t5_defer", "INDIRECT", "FIRST_NODE", {"sync": "DEFER"}),
                               ("ind_t5_chain", "INDIRECT", "FIRST_NODE", {"sync": "CHAIN"}),
                               ("ind_t1_auto", "INDIRECT", "H2D", {}),
                               ("ind_t3_auto", "INDIRECT", "ROOT_PARAMS", {}),
                               ("copy_auto", "COPY", "DEFAULT", {}),
                               ("copy_chain", "COPY", "DEFAULT", {"sync": "CHAIN"}),
                               ("setparams_auto", "SETPARAMS", "DEFAULT", {}),
                               ("ind_t5_nopdl", "INDIRECT", "FIRST_NODE", {"no_pdl": True})]:
        ex = chain.exec(mode, stream=stream, transport=xp, **kw)
        out[name] = timed(ex.handle, 2000 if cfg == "C2" else 5000)
        out[name + "_sync"] = (ex.stats()["n_deferred"], ex.stats()["dataflow"])
        ex.close()
    res[cfg] = out
    print(cfg, json.dumps(out), flush=True)
    chain.close()
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/diag_defer.json", "w"), indent=1)
