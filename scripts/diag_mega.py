"""Megakernel (persistent decoder executor) diagnostics: C3 per-replay µs of the per-node INDIRECT
graph vs the megakernel (INDIRECT, best of 3 x 200 replays), the megakernel's per-stage timeline
(CGX_MEGA_TRACE=1: first CTA start / last CTA end of every stage, µs from the first stage) and a
bitwise/tolerance comparison of the last output against the per-node exec.
Usage: diag_mega.py [T] [layers] [--fuse]"""
import json
import os
import sys

os.environ.setdefault("CGX_MEGA_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
T = int(args[0]) if args else 128
L = int(args[1]) if len(args) > 1 else 12
fuse = "--fuse" in sys.argv
dev = torch.device("cuda:0")
spec = wl.c3_chain(T=T, n_layers=L, fuse_residual=fuse)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
stream = torch.cuda.Stream()
out = {"T": T, "layers": L, "fuse": fuse}


def timeit(ex, n=200):
    for i in range(20):
        cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
        cgx.LIB.cgx_launch(ex.handle)
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for i in range(n):
            cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            cgx.LIB.cgx_launch(ex.handle)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best


last = spec.nodes[-1].out
ref = chain.exec("INDIRECT", stream=stream)
out["per_node_us"] = timeit(ref)
ref.bind({"x": xs[0]})
ref.launch()
ref_out = ref.output(last).copy()
mk = chain.exec("INDIRECT", stream=stream, megakernel=True)
out["mega_us"] = timeit(mk)
mk.bind({"x": xs[0]})
mk.launch()
mk_out = mk.output(last).copy()
out["stats"] = mk.stats()
f = lambda b: (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)  # noqa: E731
g, o = f(mk_out), f(ref_out)
out["bit_identical_to_per_node"] = bool(np.array_equal(mk_out, ref_out))
out["rel_l2_vs_per_node"] = float(np.linalg.norm(g - o) / np.linalg.norm(o))
# stage timeline of one replay: per stage the median CTA duration (start after the barrier ->
# end), the start skew over CTAs, and the barrier gap (first start of stage i+1 - last end of i)
import ctypes as C  # noqa: E402
n = cgx.LIB.cgx_debug_mega_trace(mk.handle, None, 0)
if n > 0:
    mk.bind({"x": xs[1]})
    mk.launch()
    stream.synchronize()
    buf = (C.c_uint64 * n)()
    cgx.LIB.cgx_debug_mega_trace(mk.handle, buf, n)
    ctas = 148
    arr = np.frombuffer(buf, dtype=np.uint64).astype(np.int64).reshape(-1, ctas, 8)
    n_st = arr.shape[0]
    t0 = arr[:, :, 0][arr[:, :, 0] > 0].min()
    rows = []
    prev_end = None
    for i in range(n_st):
        st_ = arr[i]
        start, end = (st_[:, 0] - t0) / 1e3, (st_[:, 1] - t0) / 1e3
        marks = {}
        for k in range(2, 7):
            m = st_[:, k] > 0
            if m.any():
                marks[k] = float(np.median((st_[m, k] - st_[m, 0]) / 1e3))
        arrive = (st_[:, 7] - t0) / 1e3
        row = {"start_min": float(start.min()), "start_max": float(start.max()), "end_max": float(end.max()),
               "dur_med": float(np.median(end - start)), "dur_max": float((end - start).max()),
               "arrive_max": float(arrive.max()) if i > 0 else 0.0,
               "release": float(start.min() - arrive.max()) if i > 0 else 0.0,
               "gap": float(start.min() - prev_end) if prev_end is not None else 0.0, "marks": marks}
        prev_end = float(end.max())
        rows.append(row)
    out["stages"] = rows
    for i, r in enumerate(rows[:10]):
        mk_ = " ".join(f"m{k}={v:5.2f}" for k, v in r["marks"].items())
        print(f"stage {i:3d} start {r['start_min']:8.2f} (+{r['start_max'] - r['start_min']:5.2f}) "
              f"dur med {r['dur_med']:5.2f} max {r['dur_max']:5.2f} | gap {r['gap']:5.2f} "
              f"(last arrival -> first release {r['release']:5.2f}) | {mk_}")
    span = max(r["end_max"] for r in rows)
    out["span_us"] = span
    print(f"span {span:.1f} us over {n_st} stages; sum of median durations {sum(r['dur_med'] for r in rows):.1f}, "
          f"sum of gaps {sum(r['gap'] for r in rows):.1f}")
print(json.dumps({k: v for k, v in out.items() if k != "stages"}))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/mega_T{T}_L{L}{'_fuse' if fuse else ''}.json", "w"))
