"""Training-shaped chain on the GPU (synth.workloads.mlp_train_chain): the init
segment copies the initial weights into INTERNAL slots once, then every replay of the step segment
runs forward, loss gradient, backward (TRANSPOSE + tcgen05 GEMMs + GELU_BWD) and the in-place SGD
update with fresh X / target. Checked per step against the oracle evaluated from the GPU's own
weights before the step; weights carried across steps; arms bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.chain import eval_chain  # noqa: E402
from oracle.numerics import bits_to_f64  # noqa: E402
from synth import workloads as wl  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _weights(spec):
    return [s.name for s in spec.slots if s.kind == "internal" and (s.name.endswith(".W1") or s.name.endswith(".W2"))]


def _train(rt, spec, mode, transport, steps):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    st = wl.static_values(spec)
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    f0, l0 = spec.segments[0]
    f1, l1 = spec.segments[1]
    init = chain.exec("EAGER", first_node=f0, n_nodes=l0 - f0 + 1)
    t0 = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    init.bind(t0)                       # (the init segment reads no external; bind takes them all)
    init.launch()
    ex = chain.exec(mode, transport=transport, first_node=f1, n_nodes=l1 - f1 + 1)
    wn = _weights(spec)
    hist, keep = [], []
    for r in range(steps):
        before = {n: ex.output(n) for n in wn}
        ext = wl.external_values(spec, r)
        t = runner.upload_externals(spec, ext, dev)
        keep.append(t)
        ex.bind(t)
        ex.launch()
        after = {s.name: ex.output(s.name) for s in spec.internals()}
        hist.append((ext, before, after))
    chain.close()
    return hist, st


@pytest.mark.parametrize("mode,transport", [("INDIRECT", "ROOT_PARAMS")])
def test_training_steps_vs_oracle(rt, mode, transport):
    spec = wl.mlp_train_chain(n_blocks=2, lr=64.0)
    hist, st = _train(rt, spec, mode, transport, 3)
    wn = _weights(spec)
    for r, (ext, before, after) in enumerate(hist):
        state = {n: bits_to_f64(before[n]) for n in wn}
        env = eval_chain(spec, ext, st, state=state, nodes=spec.segments[1])
        for name in [s.name for s in spec.internals()]:
            if name in wn:
                g, o = bits_to_f64(after[name]), env[name]
                assert np.linalg.norm(g - o) <= 2e-3 * np.linalg.norm(o), (r, name)
                continue
            if name.endswith("_0") or name not in env:       # unused slots (block 0 has no da / W1T)
                continue
            g, o = bits_to_f64(after[name]), env[name]
            no = np.linalg.norm(o)
            if no == 0:
                continue
            assert np.linalg.norm(g - o) / no <= 3e-2, (r, name, np.linalg.norm(g - o) / no)
        if r > 0:                                     # the weights carried over and changed
            prev_after = hist[r - 1][2]
            for n in wn:
                assert np.array_equal(before[n], prev_after[n])
    changed = sum(int(np.any(hist[-1][2][n] != hist[0][1][n])) for n in wn)
    assert changed == len(wn)


def test_training_arms_bitexact(rt):
    spec = wl.mlp_train_chain(n_blocks=2, lr=64.0)
    ref, _ = _train(rt, spec, "EAGER", "DEFAULT", 2)
    for mode, xp in (("INDIRECT", "FIRST_NODE"), ("INDIRECT", "ROOT_PARAMS"), ("COPY", "DEFAULT"),
                     ("SETPARAMS", "DEFAULT")):
        got, _ = _train(rt, spec, mode, xp, 2)
        for r in range(2):
            for k in ref[r][2]:
                assert np.array_equal(got[r][2][k], ref[r][2][k]), (mode, xp, r, k)
