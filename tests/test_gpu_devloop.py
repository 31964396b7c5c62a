"""NEXT-4 device-launched replays (transport DEVICE, cgx_device_loop): a scheduler
kernel binds pointer set i % n_sets into the table and tail-launches the chain graph, n_replays
times, with one host launch. Parity: every replay must see its own inputs exactly once (an
accumulating chain, integer-exact), outputs equal the oracle, host binds still work."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle import ops  # noqa: E402
from oracle.chain import eval_chain  # noqa: E402
from synth import workloads as wl  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _sets(runner, spec, n_sets, dev, mode="uniform"):
    tensors = [runner.upload_externals(spec, wl.external_values(spec, r, mode), dev) for r in range(n_sets)]
    names = [s.name for s in spec.externals()]
    table = torch.tensor([[t[n].data_ptr() for n in names] for t in tensors], dtype=torch.int64, device=dev)
    return tensors, table


@pytest.mark.parametrize("n_replays", [1, 10, 37])
def test_c1_device_loop(rt, n_replays):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="DEVICE")
    tensors, table = _sets(runner, spec, 4, dev)
    cgx.device_loop(ex.handle, table.data_ptr(), 4, n_replays)
    torch.cuda.synchronize()
    last = (n_replays - 1) % 4
    env = eval_chain(spec, wl.external_values(spec, last), st)
    for s in spec.internals():
        assert np.array_equal(ex.output(s.name), env[s.name]), s.name
    assert ex.stats()["n_launches"] == n_replays
    # the same exec still replays from host binds (H2D table path)
    ex.bind(tensors[2])
    ex.launch()
    env = eval_chain(spec, wl.external_values(spec, 2), st)
    assert np.array_equal(ex.output("out"), env["out"])
    chain.close()


def _accum_chain(n):
    s = [SlotSpec("x", "external", "f32", n), SlotSpec("acc", "internal", "f32", n),
         SlotSpec("out", "internal", "f32", n)]
    nodes = [NodeSpec("ADD", ("acc", "x"), "acc", {"n": n}), NodeSpec("COPY", ("acc",), "out", {"n": n})]
    return ChainSpec("accum", s, nodes, [(0, 1)])


@pytest.mark.parametrize("n,n_sets,n_replays", [(4096, 3, 50), (1 << 20, 5, 23)])
def test_every_replay_reads_its_own_set_once(rt, n, n_sets, n_replays):
    """acc_r = acc_{r-1} + x_{r mod n_sets}; integer-mode inputs keep every partial sum exact, so
    a replay that read a wrong or stale table entry (or ran twice / not at all) changes acc."""
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = _accum_chain(n)
    chain = runner.Chain(spec, {})
    ex = chain.exec("INDIRECT", transport="DEVICE")
    tensors, table = _sets(runner, spec, n_sets, dev, "int")
    cgx.device_loop(ex.handle, table.data_ptr(), n_sets, n_replays)
    torch.cuda.synchronize()
    acc = np.zeros(n, np.float32)
    xs = [wl.external_values(spec, r, "int")["x"] for r in range(n_sets)]
    for r in range(n_replays):
        acc = ops.add(acc, xs[r % n_sets], {"n": n})
    assert np.array_equal(ex.output("out"), acc)
    chain.close()


def test_c2_device_loop(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c2_chain()
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", transport="DEVICE")
    tensors, table = _sets(runner, spec, 3, dev)
    cgx.device_loop(ex.handle, table.data_ptr(), 3, 8)
    torch.cuda.synchronize()
    env = eval_chain(spec, wl.external_values(spec, 7 % 3), st)
    for l in range(64):
        assert np.array_equal(ex.output(f"u{l}"), env[f"u{l}"])
    chain.close()


def test_device_loop_errors(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    tensors, table = _sets(runner, spec, 2, dev)
    ex_h2d = chain.exec("INDIRECT", transport="H2D")
    with pytest.raises(cgx.CgxError):
        cgx.device_loop(ex_h2d.handle, table.data_ptr(), 2, 4)
    ex = chain.exec("INDIRECT", transport="DEVICE")
    host = table.cpu()
    with pytest.raises(cgx.CgxError):
        cgx.device_loop(ex.handle, host.data_ptr(), 2, 4)
    cgx.device_loop(ex.handle, table.data_ptr(), 2, 0)      # no-op
    torch.cuda.synchronize()
    chain.close()
