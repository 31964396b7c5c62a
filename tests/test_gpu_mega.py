"""GPU parity of the persistent decoder executor (cgx_exec_opts.megakernel): the C3
decoder chain run as ONE launch, through the C ABI against the CPU oracle.

Bar (as for the per-node decoder): every node's output slot node-local (the oracle
is fed the GPU's own node inputs) within |g - o| <= 2e-2 |o| + 2e-2 rms(o); end to end
||g - o||_2 / ||o||_2 <= 2e-2; bit-identical across the megakernel's rebinding arms (EAGER /
COPY / INDIRECT over several transports / SETPARAMS) and across replays with the same input.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from oracle.chain import eval_chain  # noqa: E402
from oracle.numerics import bits_to_f64  # noqa: E402
from synth import workloads as wl  # noqa: E402
from synth.workloads import ChainSpec, NodeSpec, SlotSpec  # noqa: E402
from test_gpu_decoder import _close, _node_local_check  # noqa: E402


@pytest.fixture(scope="module")
def rt():
    from paper_2503_19779_b200 import build
    build.build()
    from paper_2503_19779_b200 import cgx, runner
    return cgx, runner


def _run(rt, spec, mode, replays, st, **opts):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec(mode, megakernel=True, **opts)
    assert ex.stats()["kernels_per_replay"] >= 1
    outs, keep = [], []
    for r in range(replays):
        ext = wl.external_values(spec, r)
        t = runner.upload_externals(spec, ext, dev)
        keep.append(t)
        ex.bind(t)
        ex.launch()
        outs.append({s.name: ex.output(s.name) for s in spec.internals()})
    assert ex.stats()["device_error"] == 0
    chain.close()
    return outs


def _check(spec, st, outs):
    for r, got in enumerate(outs):
        ext = wl.external_values(spec, r)
        _node_local_check(spec, st, ext, got)
        env = eval_chain(spec, ext, st)
        last = spec.nodes[-1].out
        g, o = bits_to_f64(got[last]), env[last]
        assert np.linalg.norm(g - o) / np.linalg.norm(o) <= 2e-2


ARMS = [("INDIRECT", {}), ("EAGER", {}), ("COPY", {}), ("SETPARAMS", {}),
        ("INDIRECT", {"transport": "H2D"}), ("INDIRECT", {"transport": "H2D_PINGPONG"}),
        ("INDIRECT", {"transport": "PRELUDE"})]


@pytest.mark.parametrize("fuse", [False, True])
@pytest.mark.parametrize("n_layers", [1, 12])
def test_mega_c3_chain(rt, n_layers, fuse):
    spec = wl.c3_chain(T=128, n_layers=n_layers, fuse_residual=fuse)
    st = wl.static_values(spec)
    res = [_run(rt, spec, m, 2, st, **o) for m, o in ARMS]
    _check(spec, st, res[0])
    written = {n.out for n in spec.nodes}
    for (m, o), outs in zip(ARMS[1:], res[1:]):
        for r in range(2):
            for k in written:
                assert np.array_equal(outs[r][k], res[0][r][k]), (m, o, k)


@pytest.mark.parametrize("T", [1, 4, 77, 200])
def test_mega_c3_token_counts(rt, T):
    """Ragged / decode / multi-M-tile token counts (T = 200: two 128-row M tiles)."""
    spec = wl.c3_chain(T=T, n_layers=2)
    st = wl.static_values(spec)
    outs = _run(rt, spec, "INDIRECT", 2, st)
    _check(spec, st, outs)


def test_mega_matches_itself_across_replays(rt):
    """Same input bound twice: identical bits (fixed reduction orders, no atomics in the math)."""
    cgx, runner = rt
    spec = wl.c3_chain(T=128, n_layers=3)
    st = wl.static_values(spec)
    dev = torch.device("cuda:0")
    chain = runner.Chain(spec, runner.upload_statics(spec, st, dev))
    ex = chain.exec("INDIRECT", megakernel=True)
    x = runner.upload_externals(spec, wl.external_values(spec, 0), dev)
    seen = []
    for _ in range(3):
        ex.bind(x)
        ex.launch()
        seen.append(ex.output(spec.nodes[-1].out).copy())
    chain.close()
    assert all(np.array_equal(s, seen[0]) for s in seen)


def test_mega_gemm_shapes(rt):
    """LN -> GEMM (direct, K-split deferred to an ADD, and deferred at the end of the range) over
    shapes off the GPT-2 grid: N % 64 != 0, K = 320 (5 k-blocks), K needing a split to stage its weights."""
    T, d = 96, 320
    slots = [SlotSpec("x", "external", "bf16", T * d), SlotSpec("g", "static", "bf16", d, "gamma"),
             SlotSpec("b", "static", "bf16", d, "bias"), SlotSpec("ln", "internal", "bf16", T * d),
             SlotSpec("w1", "static", "bf16", 2048 * d, "weight"), SlotSpec("b1", "static", "bf16", 2048, "bias"),
             SlotSpec("f", "internal", "bf16", T * 2048),
             SlotSpec("w2", "static", "bf16", d * 2048, "weight"), SlotSpec("b2", "static", "bf16", d, "bias"),
             SlotSpec("y", "internal", "bf16", T * d), SlotSpec("z", "internal", "bf16", T * d),
             SlotSpec("w3", "static", "bf16", 96 * d, "weight"), SlotSpec("o", "internal", "bf16", T * 96)]
    nodes = [NodeSpec("LAYERNORM", ("x", "g", "b"), "ln", {"rows": T, "cols": d, "eps": 1e-5}),
             NodeSpec("GEMM_BF16", ("ln", "w1", "b1"), "f", {"M": T, "N": 2048, "K": d, "bias": True, "gelu": True}),
             NodeSpec("GEMM_BF16", ("f", "w2", "b2"), "y", {"M": T, "N": d, "K": 2048, "bias": True, "gelu": False}),
             NodeSpec("ADD", ("y", "x"), "z", {"n": T * d}),
             NodeSpec("GEMM_BF16", ("z", "w3", "b2"), "o", {"M": T, "N": 96, "K": d, "bias": False, "gelu": False})]
    spec = ChainSpec("mega_shapes", slots, nodes, [(0, 4)])
    st = wl.static_values(spec)
    for mode in ("INDIRECT", "SETPARAMS"):
        outs = _run(rt, spec, mode, 2, st)
        for r, got in enumerate(outs):
            _node_local_check(spec, st, wl.external_values(spec, r), got)


def test_mega_rejects_unsupported(rt):
    cgx, runner = rt
    dev = torch.device("cuda:0")
    spec = wl.c1_chain()                      # f32 elementwise: not a decoder range
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    with pytest.raises(RuntimeError, match="megakernel"):
        chain.exec("INDIRECT", megakernel=True)
    chain.close()
    spec = wl.c3_chain(T=128, n_layers=1)
    chain = runner.Chain(spec, runner.upload_statics(spec, wl.static_values(spec), dev))
    with pytest.raises(RuntimeError, match="FIRST_NODE"):
        chain.exec("INDIRECT", megakernel=True, transport="FIRST_NODE")
    chain.close()
