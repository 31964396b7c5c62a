"""CGX_SYNC_GRAPH (runtime.cu capture_dag): the chain captured as its data-dependency DAG over
several capture streams instead of one serial stream. Outputs must be bit-identical to the serial
capture (CHAIN) and to the oracle for every rebinding arm and transport, over many replays with
fresh input addresses, including chains with write-after-read / write-after-write hazards and
fan-in, and the decoder chain."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.chain import eval_chain  # noqa: E402
from synth import workloads as wl  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _replays(rt, spec, mode, transport, n, sync, streams=0, int_mode=False, names=None):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    vm = "int" if int_mode else "uniform"
    st = wl.static_values(spec, vm)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec(mode, transport=transport, sync=sync, graph_streams=streams)
    outs, keep = [], []
    for r in range(n):
        t = runner.upload_externals(spec, wl.external_values(spec, r, vm), dev)
        keep.append(t)
        ex.bind(t)
        ex.launch()
        outs.append({s.name: ex.output(s.name) for s in spec.internals() if names is None or s.name in names})
    chain.close()
    return outs, st


@pytest.mark.parametrize("mode,transport", [("COPY", "DEFAULT"), ("SETPARAMS", "DEFAULT"),
                                            ("INDIRECT", "H2D"), ("INDIRECT", "ROOT_MEMCPY"),
                                            ("INDIRECT", "ROOT_PARAMS"), ("INDIRECT", "ROOT_MAPPED"),
                                            ("INDIRECT", "FIRST_NODE"), ("INDIRECT", "H2D_PINGPONG")])
def test_c2_graph_sync_bitexact(rt, mode, transport):
    spec = wl.c2_chain()
    a, st = _replays(rt, spec, mode, transport, 4, "GRAPH")
    c, _ = _replays(rt, spec, mode, transport, 4, "CHAIN")
    for r in range(4):
        for k in a[r]:
            assert np.array_equal(a[r][k], c[r][k]), (mode, transport, r, k)
    env = eval_chain(spec, wl.external_values(spec, 3), st)
    for l in range(64):
        assert np.array_equal(a[3][f"t{l}"], env[f"t{l}"])
        assert np.array_equal(a[3][f"u{l}"], env[f"u{l}"])


@pytest.mark.parametrize("streams", [1, 2, 3, 8, 64])
def test_c2_graph_stream_counts(rt, streams):
    spec = wl.c2_chain(n_lanes=24)
    a, st = _replays(rt, spec, "INDIRECT", "FIRST_NODE", 3, "GRAPH", streams, int_mode=True)
    for r in (0, 2):
        env = eval_chain(spec, wl.external_values(spec, r, "int"), st)
        for k in a[r]:
            assert np.array_equal(a[r][k], env[k]), (streams, r, k)


def _hazard_chain(n):
    """RAW, WAR and WAW across lanes: t0 is read by node 1, rewritten by node 2 (WAR + WAW), and
    node 4 reads the new t0 and the old-t0 product; node 5 overwrites out (WAW) from another lane."""
    s = [SlotSpec("x0", "external", "f32", n), SlotSpec("x1", "external", "f32", n),
         SlotSpec("x2", "external", "f32", n), SlotSpec("w", "static", "f32", n),
         SlotSpec("t0", "internal", "f32", n), SlotSpec("t1", "internal", "f32", n),
         SlotSpec("t2", "internal", "f32", n), SlotSpec("out", "internal", "f32", n),
         SlotSpec("r", "internal", "f32", n // 256)]
    a = {"n": n}
    nodes = [NodeSpec("ADD", ("x0", "x1"), "t0", dict(a)),
             NodeSpec("MUL", ("t0", "x2"), "t1", dict(a)),
             NodeSpec("ADD", ("x2", "w"), "t0", dict(a)),
             NodeSpec("ADD", ("x1", "w"), "t2", dict(a)),
             NodeSpec("MUL", ("t0", "t1"), "out", dict(a)),
             NodeSpec("REDUCE_SUM", ("out",), "r", {"n": n, "cols": 256}),
             NodeSpec("MUL", ("t2", "t2"), "out", dict(a)),
             NodeSpec("ADD", ("out", "t0"), "t2", dict(a))]
    return ChainSpec("hazard", s, nodes, [(0, len(nodes) - 1)])


@pytest.mark.parametrize("n", [4096, 1 << 22])
@pytest.mark.parametrize("streams", [2, 8])
@pytest.mark.parametrize("transport", ["FIRST_NODE", "ROOT_PARAMS", "H2D"])
def test_hazards_graph_sync(rt, n, streams, transport):
    spec = _hazard_chain(n)
    outs, st = _replays(rt, spec, "INDIRECT", transport, 6, "GRAPH", streams, int_mode=True)
    for r in (0, 5):
        env = eval_chain(spec, wl.external_values(spec, r, "int"), st)
        for k in outs[r]:
            assert np.array_equal(outs[r][k], env[k]), (r, k)


def test_graph_sync_stress_rotating(rt):
    """100 replays over 4 rotating input sets (integer mode: every value exact)."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c2_chain(n_lanes=32)
    st = wl.static_values(spec, "int")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="FIRST_NODE", sync="GRAPH")
    sets = [runner.upload_externals(spec, wl.external_values(spec, r, "int"), dev) for r in range(4)]
    envs = [eval_chain(spec, wl.external_values(spec, r, "int"), st) for r in range(4)]
    names = [f"r{l}" for l in range(32)]
    for i in range(100):
        ex.bind(sets[i % 4])
        ex.launch()
        if i % 7 == 0 or i >= 96:
            for nm in names:
                assert np.array_equal(ex.output(nm), envs[i % 4][nm]), (i, nm)
    chain.close()


def test_c3_decoder_graph_sync_bitexact(rt):
    spec = wl.c3_chain(T=128, n_layers=2)
    names = {s.name for s in spec.internals()}
    a, _ = _replays(rt, spec, "INDIRECT", "FIRST_NODE", 2, "GRAPH", names=names)
    c, _ = _replays(rt, spec, "INDIRECT", "FIRST_NODE", 2, "CHAIN", names=names)
    for r in range(2):
        for k in a[r]:
            assert np.array_equal(a[r][k], c[r][k]), (r, k)


@pytest.mark.parametrize("transport", ["PRELUDE", "DEVICE"])
def test_graph_sync_prelude_and_device_transports(rt, transport):
    """The opaque-kernel prelude (device-side param updates before the fork) and the device-launched
    replay loop on the DAG capture: bit-identical to the serial dataflow capture and the oracle."""
    cgx, runner = rt
    spec = wl.c2_chain(n_lanes=20)
    if transport == "PRELUDE":
        a, st = _replays(rt, spec, "INDIRECT", transport, 3, "GRAPH", int_mode=True)
        c, _ = _replays(rt, spec, "INDIRECT", transport, 3, "DATAFLOW", int_mode=True)
        for r in range(3):
            env = eval_chain(spec, wl.external_values(spec, r, "int"), st)
            for k in a[r]:
                assert np.array_equal(a[r][k], c[r][k]) and np.array_equal(a[r][k], env[k]), (r, k)
        return
    dev = torch.device("cuda:0")
    st = wl.static_values(spec, "int")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="DEVICE", sync="GRAPH")
    sets = [runner.upload_externals(spec, wl.external_values(spec, r, "int"), dev) for r in range(3)]
    names = [s_.name for s_ in spec.externals()]
    ptrs = torch.tensor([[t[n].data_ptr() for n in names] for t in sets], dtype=torch.int64, device=dev)
    cgx.device_loop(ex.handle, ptrs.data_ptr(), 3, 5)      # replays 0..4 bind sets 0,1,2,0,1
    torch.cuda.synchronize()
    env = eval_chain(spec, wl.external_values(spec, 1, "int"), st)
    for l in range(20):
        assert np.array_equal(ex.output(f"r{l}"), env[f"r{l}"]), l
    chain.close()


@pytest.mark.parametrize("order", ["priority", "level"])
def test_graph_sync_issue_orders(rt, order, monkeypatch):
    """Any topological issue order (CGX_DAG_ORDER, read at capture) gives the oracle's results."""
    monkeypatch.setenv("CGX_DAG_ORDER", order)
    for spec in (wl.c2_chain(n_lanes=24), _hazard_chain(4096)):
        a, st = _replays(rt, spec, "INDIRECT", "FIRST_NODE", 3, "GRAPH", int_mode=True)
        for r in (0, 2):
            env = eval_chain(spec, wl.external_values(spec, r, "int"), st)
            for k in a[r]:
                assert np.array_equal(a[r][k], env[k]), (order, r, k)


def test_tune_graph_streams(rt):
    """cgx_tune_graph_streams (slow path): measures each candidate stream count on the given
    inputs and returns the fastest; the exec deployed with it is bit-exact; EAGER is rejected."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c2_chain(n_lanes=24)
    st = wl.static_values(spec, "int")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    sets = [runner.upload_externals(spec, wl.external_values(spec, r, "int"), dev) for r in range(2)]
    ptrs = [[t[n].data_ptr() for n in chain.ext_names] for t in sets]
    stream = torch.cuda.current_stream()
    best, us = cgx.tune_graph_streams(chain.handle, "INDIRECT", stream.cuda_stream, ptrs, candidates=(2, 8, 16),
                                      reps=20, transport="ROOT_PARAMS")
    assert best in (2, 8, 16) and set(us) == {2, 8, 16}
    assert all(v > 0 for v in us.values()) and us[best] == min(us.values())
    with pytest.raises(cgx.CgxError):
        cgx.tune_graph_streams(chain.handle, "EAGER", stream.cuda_stream, ptrs, candidates=(2,), reps=2)
    ex = chain.exec("INDIRECT", transport="ROOT_PARAMS", graph_streams=best)
    ex.bind(sets[1])
    ex.launch()
    env = eval_chain(spec, wl.external_values(spec, 1, "int"), st)
    for l in range(24):
        assert np.array_equal(ex.output(f"r{l}"), env[f"r{l}"]), l
    chain.close()
