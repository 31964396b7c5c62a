import sys, json, torch
sys.path.insert(0, ".")
from paper_2503_19779_b200 import cgx, runner
from synth import workloads as wl
dev = torch.device("cuda:0"); stream = torch.cuda.Stream()
spec = wl.mlp_train_chain(n_blocks=6)
chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
f0, l0 = spec.segments[0]; f1, l1 = spec.segments[1]
sets = [runner.upload_externals(spec, wl.external_values(spec, r), dev) for r in range(4)]
ptrs = [cgx.ptr_array([t[n].data_ptr() for n in chain.ext_names]) for t in sets]
L = cgx.LIB
init = chain.exec("EAGER", stream=stream, first_node=f0, n_nodes=l0 - f0 + 1)
L.cgx_bind(init.handle, ptrs[0], 2); L.cgx_launch(init.handle)
def timed(h, n):
    best = 1e30
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        stream.synchronize(); e0.record(stream)
        for i in range(n):
            L.cgx_bind(h, ptrs[i % 4], 2); L.cgx_launch(h)
        e1.record(stream); e1.synchronize(); best = min(best, e0.elapsed_time(e1) * 1e3 / n)
    return best
for mode, xp, sync in (("INDIRECT","ROOT_PARAMS","AUTO"),("INDIRECT","H2D","AUTO"),("INDIRECT","FIRST_NODE","AUTO"),("COPY","DEFAULT","AUTO"),("SETPARAMS","DEFAULT","AUTO"),
                       ("INDIRECT","ROOT_PARAMS","CHAIN"),("COPY","DEFAULT","CHAIN")):
    ex = chain.exec(mode, stream=stream, transport=xp, first_node=f1, n_nodes=l1 - f1 + 1, sync=sync)
    for i in range(5): L.cgx_bind(ex.handle, ptrs[i % 4], 2); L.cgx_launch(ex.handle)
    st = ex.stats()
    print(json.dumps({"mode": mode, "xport": xp, "sync": sync, "us": timed(ex.handle, 100), "dag_streams": st["dag_streams"], "graph_nodes": st["n_graph_nodes"]}), flush=True)
    ex.close()
