"""Diagnostic: launch cadence of the library's own chain kernels in a PDL graph (dataflow mode).
Chains of 200 nodes: (a) independent ADD(x_i, w_i) -> t_i (no dependencies), (b) a linear chain
t_{i} = ADD(t_{i-1}, w_i), (c) lanes of ADD->MUL->REDUCE at a fixed size; sizes 1 KiB / 64 KiB."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_19779_b200 import build  # noqa: E402

build.build()
from paper_2503_19779_b200 import cgx, runner  # noqa: E402
from synth import workloads as wl  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream()


def indep(n, K=200):
    s, nodes = [], []
    for i in range(K):
        s += [SlotSpec(f"x{i}", "external", "f32", n), SlotSpec(f"w{i}", "static", "f32", n),
              SlotSpec(f"t{i}", "internal", "f32", n)]
        nodes.append(NodeSpec("ADD", (f"x{i}", f"w{i}"), f"t{i}", {"n": n}))
    return ChainSpec("indep", s, nodes, [(0, K - 1)])


def linear(n, K=200):
    s = [SlotSpec("x", "external", "f32", n)] + [SlotSpec(f"w{i}", "static", "f32", n) for i in range(K)]
    s += [SlotSpec(f"t{i}", "internal", "f32", n) for i in range(K)]
    nodes = [NodeSpec("ADD", ("x" if i == 0 else f"t{i-1}", f"w{i}"), f"t{i}", {"n": n}) for i in range(K)]
    return ChainSpec("linear", s, nodes, [(0, K - 1)])


def lanes(n, L=66):
    s, nodes = [], []
    for l in range(L):
        s += [SlotSpec(f"x{l}", "external", "f32", n), SlotSpec(f"w{l}", "static", "f32", n),
              SlotSpec(f"t{l}", "internal", "f32", n), SlotSpec(f"u{l}", "internal", "f32", n),
              SlotSpec(f"r{l}", "internal", "f32", n // 256)]
        nodes += [NodeSpec("ADD", (f"x{l}", f"w{l}"), f"t{l}", {"n": n}),
                  NodeSpec("MUL", (f"t{l}", f"x{l}"), f"u{l}", {"n": n}),
                  NodeSpec("REDUCE_SUM", (f"u{l}",), f"r{l}", {"n": n, "cols": 256})]
    return ChainSpec("lanes", s, nodes, [(0, len(nodes) - 1)])


res = {}
for name, mk in (("indep", indep), ("linear", linear), ("lanes", lanes)):
    for nb in (1024, 65536):
        spec = mk(nb // 4)
        chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
        sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(4)]
        ptrs = [cgx.ptr_array([t[n_].data_ptr() for n_ in chain.ext_names]) for t in sets]
        for sync in ("AUTO", "CHAIN"):
            ex = chain.exec("INDIRECT", stream=stream, transport="H2D", sync=sync)
            N = 500

            def go():
                for i in range(N):
                    cgx.LIB.cgx_bind(ex.handle, ptrs[i % 4], len(chain.ext_names))
                    cgx.LIB.cgx_launch(ex.handle)
            go()
            best = 1e9
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                stream.synchronize()
                with torch.cuda.stream(stream):
                    e0.record(stream)
                    go()
                    e1.record(stream)
                e1.synchronize()
                best = min(best, e0.elapsed_time(e1) * 1e3 / N)
            key = f"{name}_{nb}B_{sync}"
            res[key] = {"us_per_replay": best, "us_per_node": best / len(spec.nodes)}
            print(key, json.dumps(res[key]), flush=True)
            ex.close()
        chain.close()
print("graph_floor_200_pdl_nop", cgx.graph_floor(stream.cuda_stream, 200, True, 300) / 200)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/diag_cadence.json", "w"), indent=1)
