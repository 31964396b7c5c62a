"""Sweep the decoder GEMM's operand grouping / tiling knobs (CGX_GEMM_GROUP, CGX_GEMM_RING,
CGX_GEMM_TILING) on the real objective: the deployed 12-layer C3 replay (INDIRECT, T=128, µs per
replay, best of 3 x 200), plus the standalone per-shape GEMM span from the phase tracer.
Each configuration runs in a child process (the knobs are read at exec build time)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_2503_19779_b200 import cgx, runner
    from synth import workloads as wl
    dev = torch.device("cuda:0")
    out = {}
    spec = wl.c3_chain(T=128, n_layers=12)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    xs = [runner.host_to_device(wl.slot_values(spec, "x", r), "bf16", dev) for r in range(4)]
    ptrs = [cgx.ptr_array([x.data_ptr()]) for x in xs]
    stream = torch.cuda.Stream()
    ex = chain.exec("INDIRECT", stream=stream)
    LIB = cgx.LIB
    for i in range(20):
        LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
        LIB.cgx_launch(ex.handle)
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize()
        e0.record(stream)
        for i in range(200):
            LIB.cgx_bind(ex.handle, ptrs[i % 4], 1)
            LIB.cgx_launch(ex.handle)
        e1.record(stream)
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / 200)
    out["c3_us"] = round(best, 1)
    ex.close()
    chain.close()
    spec = wl.c3_chain(T=128, n_layers=1)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec("COPY")
    x = runner.host_to_device(wl.slot_values(spec, "x", 0), "bf16", dev)
    ex.bind({"x": x})
    ex.launch()
    torch.cuda.synchronize()
    for pos, node in enumerate(spec.nodes):
        if node.op != "GEMM_BF16":
            continue
        spans, phases = [], []
        names = ["entry", "setup", "stage0", "mma_issued", "stored", "pushed", "arrived", "exit", "acc_ready",
                 "acc_regs", "staged", "a_issued", "refill_ok", "mma_at_refill", "refill_landed", "mma_last"]
        for rep in range(6):
            tr = np.array(cgx.gemm_trace(ex.handle, pos), dtype=np.float64)
            t0 = tr[:, 0].min()
            spans.append((tr[:, 7].max() - t0) / 1e3)
            rel = (tr - t0) / 1e3
            rel[tr == 0] = np.nan
            phases.append([float(np.nanmedian(rel[:, i])) if not np.all(np.isnan(rel[:, i])) else None
                           for i in range(len(names))])
        a = node.attrs
        med = {nm: (round(float(np.median([p[i] for p in phases[1:]])), 2) if phases[1][i] is not None else None)
               for i, nm in enumerate(names)}
        out[f"{a['N']}x{a['K']}"] = {"ctas": len(tr), "span": round(float(np.median(spans[1:])), 2),
                                     "phase_med_us": {k: v for k, v in med.items() if v is not None}}
    print(json.dumps(out))
    chain.close()
else:
    configs = [c.split(";") for c in (sys.argv[1:] or [
        "", "CGX_GEMM_GROUP=1;CGX_GEMM_RING=4", "CGX_GEMM_GROUP=1", "CGX_GEMM_GROUP=2", "CGX_GEMM_GROUP=3",
        "CGX_GEMM_GROUP=2;CGX_GEMM_RING=2", "CGX_GEMM_GROUP=3;CGX_GEMM_RING=2"])]
    for cfg in configs:
        env = dict(os.environ)
        for kv in cfg:
            if kv:
                k, v = kv.split("=", 1)
                env[k] = v
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True, timeout=300)
        print(json.dumps({"cfg": ";".join(cfg) or "default", "res": (json.loads(r.stdout.strip().splitlines()[-1])
                                                                     if r.returncode == 0 else r.stderr[-800:])}),
              flush=True)
