"""COPY-arm Δ on C2 for several copy-kernel grid sizes (CGX_COPY_CTAS knob) + kernel_times sanity."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2503_19779_b200 import cgx, runner
    from synth import splitmix as sm, workloads as wl
    dev = torch.device("cuda:0"); stream = torch.cuda.Stream(); sh = stream.cuda_stream; LIB = cgx.LIB
    spec = wl.c2_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ext = spec.externals(); sets = []
    for r in range(8):
        ts = [torch.empty(s.nelems, dtype=torch.float32, device=dev) for s in ext]
        for s, t in zip(ext, ts):
            cgx.fill_uniform_f32(t.data_ptr(), s.nelems, sm.SEED, sm.stream_id(spec.index(s.name), r), sh)
        sets.append((ts, cgx.ptr_array([t.data_ptr() for t in ts])))
    torch.cuda.synchronize()
    ex = chain.exec("COPY", stream=stream)
    def timed(bind, n=2000):
        for i in range(10):
            LIB.cgx_bind(ex.handle, sets[i % 8][1], 64); LIB.cgx_launch(ex.handle)
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize(); e0.record(stream)
            for i in range(n):
                if bind: LIB.cgx_bind(ex.handle, sets[i % 8][1], 64)
                LIB.cgx_launch(ex.handle)
            e1.record(stream); e1.synchronize(); best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        return best
    b = timed(False); c = timed(True)
    # copy kernel alone
    ds = []
    for i in range(50):
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize(); a0.record(stream); LIB.cgx_bind(ex.handle, sets[i % 8][1], 64); a1.record(stream); a1.synchronize()
        ds.append(a0.elapsed_time(a1) * 1e3)
    kt = cgx.kernel_times(ex.handle, 50)
    print(json.dumps({"ctas": os.environ.get("CGX_COPY_CTAS"), "base": b, "copy": c, "delta": c - b,
                      "copy_kernel_us_mean": sum(ds) / len(ds), "sum_kernel_times": sum(kt),
                      "kt_first8": kt[:8]}))
else:
    for ctas in ["296", "592", "1184", "2368"]:
        env = dict(os.environ, CGX_COPY_CTAS=ctas)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-2000:], flush=True)
