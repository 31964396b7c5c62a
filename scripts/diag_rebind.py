"""Diagnostics: where does each arm's rebinding cost go? (device-timeline µs per replay)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_19779_b200 import build
build.build()
from paper_2503_19779_b200 import cgx, runner
from synth import splitmix as sm, workloads as wl

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
    n_ext = len(ext)

    def timed(h, n, bind=True):
        for i in range(10):
            if bind: LIB.cgx_bind(h, sets[i % R][1], n_ext)
            LIB.cgx_launch(h)
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(n):
                if bind:
                    assert LIB.cgx_bind(h, sets[i % R][1], n_ext) == 0, cgx.last_error()
                assert LIB.cgx_launch(h) == 0, cgx.last_error()
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        return best
    N = 2000 if cfg == "C2" else 5000
    out = {}
    for name, mode, xp, nopdl in [("copy", "COPY", "DEFAULT", False), ("copy_nopdl", "COPY", "DEFAULT", True),
                                  ("t1", "INDIRECT", "H2D", False), ("t2", "INDIRECT", "ROOT_MEMCPY", False),
                                  ("t3", "INDIRECT", "ROOT_PARAMS", False), ("t4", "INDIRECT", "ROOT_MAPPED", False), ("t5", "INDIRECT", "FIRST_NODE", False), ("t6", "INDIRECT", "H2D_PINGPONG", False),
                                  ("t3_nopdl", "INDIRECT", "ROOT_PARAMS", True), ("setparams", "SETPARAMS", "DEFAULT", False),
                                  ("eager", "EAGER", "DEFAULT", False)]:
        ex = chain.exec(mode, stream=stream, transport=xp, no_pdl=nopdl)
        n = N if mode != "EAGER" else 200
        out[name + "_bind_launch"] = timed(ex.handle, n, True)
        if mode not in ("EAGER",):
            out[name + "_launch_only"] = timed(ex.handle, n, False)
        ex.close()
    for nk in (1, 8, 200):
        out[f"graph_floor_{nk}_pdl"] = cgx.graph_floor(sh, nk, True, 500)
        out[f"graph_floor_{nk}_nopdl"] = cgx.graph_floor(sh, nk, False, 500)
    g, k = cgx.dispatch_floor(sh, 2000)
    out["floor_graph_launch_host_us"] = g
    out["floor_kernel_launch_host_us"] = k
    res[cfg] = out
    chain.close()
print(json.dumps(res, indent=1))

# ---- copy kernel variants at the C4 1 GiB point (bind = copy only)
S = 1 << 30
c4 = wl.c4_chain(S, window_mode=True)
ch = runner.Chain(c4, runner.upload_statics(c4, wl.static_values(c4), dev))
srcs = [torch.empty(S // 4, dtype=torch.float32, device=dev) for _ in range(3)]
for i, t in enumerate(srcs):
    cgx.fill_uniform_f32(t.data_ptr(), S // 4, sm.SEED, i, sh)
arr = cgx.ptr_array([t.data_ptr() for t in srcs])
cres = {}
for impl in (0, 2, 1):
    ex = ch.exec("COPY", stream=stream, copy_impl=impl)
    ds = []
    for i in range(12):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        a.record(stream)
        LIB.cgx_bind(ex.handle, arr, 3)
        b.record(stream)
        b.synchronize()
        if i >= 2:
            ds.append(a.elapsed_time(b) * 1e-3)
    dt = statistics.median(ds)
    cres[f"impl{impl}"] = {"us": dt * 1e6, "GBps": 6 * S / dt / 1e9}
    ex.close()
t = torch.empty(3 * S // 2, dtype=torch.bfloat16, device=dev)
u = torch.empty_like(t)
ds = []
for i in range(12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); u.copy_(t); b.record(); b.synchronize()
    if i >= 2: ds.append(a.elapsed_time(b) * 1e-3)
cres["torch_copy_3GiB"] = {"GBps": 2 * 3 * S / statistics.median(ds) / 1e9}
print(json.dumps({"copy_1GiBx3": cres}, indent=1))
