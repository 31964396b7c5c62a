"""Node synchronisation modes in graph replays: DATAFLOW (per-node completion counters), DEFER
(deferred griddepcontrol.wait for nodes with no in-graph producer) and CHAIN (plain PDL waits).
Outputs must be bit-identical across modes, to EAGER and to the oracle, over many replays with
fresh input addresses, including chains with write-after-read / write-after-write hazards."""
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


def _replays(rt, spec, mode, transport, n, sync, int_mode=False):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    st = wl.static_values(spec, "int" if int_mode else "uniform")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec(mode, transport=transport, sync=sync)
    outs, keep = [], []
    for r in range(n):
        vals = wl.external_values(spec, r, "int" if int_mode else "uniform")
        t = runner.upload_externals(spec, vals, dev)
        keep.append(t)
        ex.bind(t)
        ex.launch()
        outs.append({s.name: ex.output(s.name) for s in spec.internals()})
    stt = ex.stats()
    chain.close()
    return outs, (stt["n_deferred"], stt["dataflow"]), st


@pytest.mark.parametrize("transport,want", [("FIRST_NODE", 64), ("H2D", 64), ("ROOT_PARAMS", 63)])
def test_c2_sync_modes_bitexact(rt, transport, want):
    spec = wl.c2_chain()
    a, sa, st = _replays(rt, spec, "INDIRECT", transport, 6, "DATAFLOW")
    b, sb, _ = _replays(rt, spec, "INDIRECT", transport, 6, "DEFER")
    c, sc, _ = _replays(rt, spec, "INDIRECT", transport, 6, "CHAIN")
    assert sa == (0, 1) and sb == (want, 0) and sc == (0, 0)
    for r in range(6):
        for k in a[r]:
            assert np.array_equal(a[r][k], c[r][k]), (r, k)
            assert np.array_equal(b[r][k], c[r][k]), (r, k)
    env = eval_chain(spec, wl.external_values(spec, 5), st)
    for l in range(64):
        assert np.array_equal(a[5][f"t{l}"], env[f"t{l}"])
        assert np.array_equal(a[5][f"u{l}"], env[f"u{l}"])


@pytest.mark.parametrize("mode", ["COPY", "SETPARAMS", "EAGER", "STALE"])
def test_c2_sync_other_modes(rt, mode):
    spec = wl.c2_chain(n_lanes=16)
    a, sa, _ = _replays(rt, spec, mode, "DEFAULT", 4, "DATAFLOW")
    b, sb, _ = _replays(rt, spec, mode, "DEFAULT", 4, "DEFER")
    c, _, _ = _replays(rt, spec, mode, "DEFAULT", 4, "CHAIN")
    graph = mode != "EAGER"                       # eager keeps the wait: previous iteration
    assert sa == ((0, 1) if graph else (0, 0)) and sb == ((16, 0) if graph else (0, 0))
    for r in range(4):
        for k in a[r]:
            assert np.array_equal(a[r][k], c[r][k])
            assert np.array_equal(b[r][k], c[r][k])


def _war_chain(n):
    s = [SlotSpec("x0", "external", "f32", n), SlotSpec("x1", "external", "f32", n),
         SlotSpec("x2", "external", "f32", n), SlotSpec("w", "static", "f32", n),
         SlotSpec("t0", "internal", "f32", n), SlotSpec("t1", "internal", "f32", n),
         SlotSpec("t2", "internal", "f32", n), SlotSpec("out", "internal", "f32", n)]
    a = {"n": n}
    nodes = [NodeSpec("ADD", ("x0", "x1"), "t0", dict(a)),       # deferrable (nothing earlier)
             NodeSpec("MUL", ("t0", "x2"), "t1", dict(a)),       # reads t0
             NodeSpec("ADD", ("x2", "w"), "t0", dict(a)),        # WAR on t0: must keep its wait
             NodeSpec("ADD", ("x1", "w"), "t2", dict(a)),        # deferrable
             NodeSpec("MUL", ("t0", "t1"), "out", dict(a))]
    return ChainSpec("war", s, nodes, [(0, 4)])


@pytest.mark.parametrize("n", [4096, 1 << 22])
@pytest.mark.parametrize("sync,want", [("DATAFLOW", (0, 1)), ("DEFER", (2, 0))])
def test_war_hazard(rt, n, sync, want):
    spec = _war_chain(n)
    outs, got, st = _replays(rt, spec, "INDIRECT", "FIRST_NODE", 8, sync)
    assert got == want               # DEFER: node 2 rewrites t0 (read by node 1) -> keeps its wait
    for r in (0, 7):
        env = eval_chain(spec, wl.external_values(spec, r), st)
        for k in ("t0", "t1", "t2", "out"):
            assert np.array_equal(outs[r][k], env[k]), (r, k)


def _fanin_chain(n, readers):
    """One slot read by many nodes, then overwritten: the writer's WAR set exceeds the dataflow
    dependency cap, so the exec falls back to deferred waits."""
    s = [SlotSpec("x", "external", "f32", n), SlotSpec("w", "static", "f32", n),
         SlotSpec("t", "internal", "f32", n)] + [SlotSpec(f"o{i}", "internal", "f32", n) for i in range(readers)]
    a = {"n": n}
    nodes = [NodeSpec("ADD", ("x", "w"), "t", dict(a))]
    nodes += [NodeSpec("MUL", ("t", "x"), f"o{i}", dict(a)) for i in range(readers)]
    nodes += [NodeSpec("ADD", ("x", "x"), "t", dict(a)), NodeSpec("MUL", ("t", "o0"), "o0", dict(a))]
    return ChainSpec("fanin", s, nodes, [(0, len(nodes) - 1)])


@pytest.mark.parametrize("readers,df", [(3, 1), (6, 0)])
def test_fanin_fallback(rt, readers, df):
    spec = _fanin_chain(1 << 16, readers)
    outs, got, st = _replays(rt, spec, "INDIRECT", "FIRST_NODE", 4, "DATAFLOW")
    assert got[1] == df
    env = eval_chain(spec, wl.external_values(spec, 3), st)
    for k in outs[3]:
        assert np.array_equal(outs[3][k], env[k]), k


@pytest.mark.parametrize("sync", ["DATAFLOW", "DEFER"])
def test_c2_sync_stress_rotating(rt, sync):
    """100 replays over 4 rotating input sets (integer mode: every value exact)."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c2_chain(n_lanes=32)
    st = wl.static_values(spec, "int")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="FIRST_NODE", sync=sync)
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
