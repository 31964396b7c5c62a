"""C3 decoder replay (12 layers, T = 128, INDIRECT, best of 3 x 300 replays with 4 rotating inputs)
under measurement knobs set in the environment of a child process per configuration (the knobs are
read at exec build time): CGX_LN_WARPS, CGX_ATTN_WARPS, CGX_GEMM_TILING, ...
Usage: sweep_c3_knobs.py "ENV=V[;ENV2=V2]" ...   (an empty string = defaults)"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import torch
    from paper_2503_19779_b200 import cgx, runner
    from synth import workloads as wl
    dev = torch.device("cuda:0")
    stream = torch.cuda.Stream()
    res = {}
    for fuse in (False, True, "add_ln", "ln_gemm"):
        spec = wl.c3_chain(T=128, n_layers=12, fuse_residual=fuse is True or fuse == "ln_gemm")
        chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
        xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
        ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
        ex = chain.exec("INDIRECT", stream=stream, fuse=cgx.FUSE_ADD_LN if fuse == "add_ln" else
                        cgx.FUSE_LN_GEMM if fuse == "ln_gemm" else 0)
        for i in range(30):
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
        res[fuse if isinstance(fuse, str) else "fused" if fuse else "unfused"] = round(best, 1)
        chain.close()
    print(json.dumps(res))
    sys.exit(0)

sys.path.insert(0, ROOT)
from paper_2503_19779_b200 import build  # noqa: E402
build.build()
for cfg in sys.argv[1:] or [""]:
    env = dict(os.environ)
    for kv in filter(None, cfg.split(";")):
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=300)
    line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else r.stderr[-300:]
    print(json.dumps({"cfg": cfg or "default", "res": line}), flush=True)
