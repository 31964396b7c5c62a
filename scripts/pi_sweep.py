"""E5 analog (fig:triton-non-triton-indirection-overheads): rebinding cost vs
number of indirected parameters, in-kernel dereference (PI for rewritable kernels) vs the prelude
kernel (PI for opaque kernels, NEXT-1), plus the other arms for reference.

Chain: P nodes t_i = ADD(x_i, w) over 1024 fp32, one external pointer per node (P params).
Δ = device-timeline µs per replay (bind + launch, 2000 back-to-back replays, best of 3) minus the
same graph replayed with no rebinding at all.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import splitmix as sm  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
sh = stream.cuda_stream
LIB = cgx.LIB
N = 1024
res = {}
for P in (1, 2, 4, 8, 16, 32, 64, 128, 256):
    slots = [SlotSpec("w", "static", "f32", N)] + [SlotSpec(f"x{i}", "external", "f32", N) for i in range(P)] + \
            [SlotSpec(f"t{i}", "internal", "f32", N) for i in range(P)]
    nodes = [NodeSpec("ADD", (f"x{i}", "w"), f"t{i}", {"n": N}) for i in range(P)]
    spec = ChainSpec(f"pi{P}", slots, nodes, [(0, P - 1)])
    w = torch.empty(N, dtype=torch.float32, device=dev)
    cgx.fill_uniform_f32(w.data_ptr(), N, sm.SEED, 1, sh)
    chain = runner.Chain(spec, {"w": w})
    sets = []
    for r in range(4):
        ts = [torch.empty(N, dtype=torch.float32, device=dev) for _ in range(P)]
        for i, t in enumerate(ts):
            cgx.fill_uniform_f32(t.data_ptr(), N, sm.SEED, (i << 20) | r, sh)
        sets.append((ts, cgx.ptr_array([t.data_ptr() for t in ts])))
    torch.cuda.synchronize()

    def timed(h, bind, n=2000):
        for i in range(10):
            LIB.cgx_bind(h, sets[i % 4][1], P)
            LIB.cgx_launch(h)
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            stream.synchronize()
            e0.record(stream)
            for i in range(n):
                if bind:
                    assert LIB.cgx_bind(h, sets[i % 4][1], P) == 0, cgx.last_error()
                assert LIB.cgx_launch(h) == 0, cgx.last_error()
            e1.record(stream)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e3 / n)
        return best
    out = {}
    exc = chain.exec("COPY", stream=stream)
    base = timed(exc.handle, False)
    out["graph_no_rebind_us"] = base
    out["copy"] = timed(exc.handle, True) - base
    exc.close()
    for name, mode, xp in (("indirect_in_kernel_h2d", "INDIRECT", "H2D"),
                           ("indirect_in_kernel_pingpong", "INDIRECT", "H2D_PINGPONG"),
                           ("indirect_in_kernel_first_node", "INDIRECT", "FIRST_NODE"),
                           ("indirect_prelude", "INDIRECT", "PRELUDE"),
                           ("setparams", "SETPARAMS", "DEFAULT")):
        try:
            ex = chain.exec(mode, stream=stream, transport=xp)
            out[name] = timed(ex.handle, True) - base
            ex.close()
        except cgx.CgxError as exn:
            out[name] = str(exn)
    res[P] = out
    print(P, json.dumps(out), flush=True)
    chain.close()
json.dump(res, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out",
                                 "pi_sweep.json"), "w"), indent=1)
