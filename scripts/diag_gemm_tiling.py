"""Compare GEMM tilings (N tile x split-K) per decoder shape: kernel span from the phase tracer."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    import numpy as np, torch
    from paper_2503_19779_b200 import cgx, runner
    from synth import workloads as wl
    dev = torch.device("cuda:0")
    spec = wl.c3_chain(T=128, n_layers=1)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    ex = chain.exec("COPY")
    x = runner.host_to_device(wl.slot_values(spec, "x", 0), "bf16", dev)
    ex.bind({"x": x}); ex.launch(); torch.cuda.synchronize()
    out = {}
    for pos, node in enumerate(spec.nodes):
        if node.op != "GEMM_BF16":
            continue
        spans = []
        for rep in range(6):
            tr = np.array(cgx.gemm_trace(ex.handle, pos), dtype=np.float64)
            spans.append((tr[:, 7].max() - tr[:, 0].min()) / 1e3)
        a = node.attrs
        out[f"{a['M']}x{a['N']}x{a['K']}"] = {"ctas": len(tr), "span_us_med": float(np.median(spans[1:]))}
    print(json.dumps(out))
    chain.close()
else:
    # default (model-picked) tiling first, then forced (BN, split) pairs
    combos = [(None, None)] + [(bn, sp) for bn in ("32", "64", "128") for sp in ("1", "2", "3", "4", "6", "8")]
    for bn, sp in combos:
        env = dict(os.environ)
        if bn:
            env.update(CGX_GEMM_BN=bn, CGX_GEMM_SPLIT=sp)
        r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True)
        print(f"BN={bn or 'model'} split={sp or 'model'}", (r.stdout.strip() or r.stderr[-600:]), flush=True)
