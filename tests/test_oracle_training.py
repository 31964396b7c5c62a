"""Pins for the training-shaped chain's oracle (synth.workloads.mlp_train_chain):
the backward pass and the SGD update are checked against a finite-difference gradient of the loss
computed by an independent float64 forward pass (plain NumPy matmuls, no bf16 rounding), and the
op definitions against closed forms."""
import math

import numpy as np
import pytest

from oracle import ops
from oracle.chain import eval_chain
from oracle.numerics import bits_to_f64
from synth import workloads as wl


def test_gelu_grad_is_the_derivative():
    x = np.linspace(-5, 5, 201)
    h = 1e-6
    num = (ops.gelu_tanh(x + h) - ops.gelu_tanh(x - h)) / (2 * h)
    assert np.max(np.abs(num - ops.gelu_grad(x))) < 1e-8
    assert ops.gelu_grad(np.array([0.0]))[0] == 0.5                      # GELU'(0) = 1/2


def test_transpose_sub_axpy_closed_forms():
    a = np.arange(12, dtype=np.float64)
    t = ops.transpose(a, {"n": 12, "cols": 4})
    assert np.array_equal(t.reshape(4, 3), a.reshape(3, 4).T)
    assert np.array_equal(ops.transpose(t, {"n": 12, "cols": 3}), a)     # involution
    b = np.full(12, 2.0)
    assert np.array_equal(ops.sub(a, b, {"n": 12}), a - 2.0)
    assert np.array_equal(ops.axpy(a, b, {"n": 12, "scalar": -0.5}), a - 1.0)


def _forward_loss(blocks, X, target):
    a = X
    for W1, W2 in blocks:
        a = ops.gelu_tanh(a @ W1.T) @ W2.T
    return float(np.mean((a - target) ** 2))


@pytest.mark.parametrize("n_blocks", [1, 2])
def test_backward_matches_finite_differences(n_blocks):
    T, d, dff = 4, 8, 16
    spec = wl.mlp_train_chain(T=T, d=d, dff=dff, n_blocks=n_blocks, lr=1.0)
    st = wl.static_values(spec)
    ext = wl.external_values(spec, 0)
    init = eval_chain(spec, ext, st, nodes=spec.segments[0])
    state = {k: v for k, v in init.items() if k.endswith(".W1") or k.endswith(".W2")}
    env = eval_chain(spec, ext, st, state=state, nodes=spec.segments[1])
    X = bits_to_f64(ext["X"]).reshape(T, d)
    target = bits_to_f64(ext["target"]).reshape(T, d)
    blocks = [(state[f"B{l}.W1"].reshape(dff, d), state[f"B{l}.W2"].reshape(d, dff)) for l in range(n_blocks)]
    eps = 1e-4
    rng = np.random.default_rng(0)
    for l in range(n_blocks):
        for name, shape, idx in (("dW1", (dff, d), 0), ("dW2", (d, dff), 1)):
            g = env[f"B{l}.{name}"].reshape(shape)
            for _ in range(6):
                i, j = rng.integers(shape[0]), rng.integers(shape[1])
                plus = [list(b) for b in blocks]
                minus = [list(b) for b in blocks]
                plus[l][idx] = blocks[l][idx].copy()
                minus[l][idx] = blocks[l][idx].copy()
                plus[l][idx][i, j] += eps
                minus[l][idx][i, j] -= eps
                num = (_forward_loss(plus, X, target) - _forward_loss(minus, X, target)) / (2 * eps)
                scale = np.max(np.abs(g)) + 1e-30
                assert abs(g[i, j] - num) <= 3e-2 * scale, (l, name, i, j, g[i, j], num)
    # the SGD step: W_new = bf16(W - lr * dW)
    for l in range(n_blocks):
        for w in ("W1", "W2"):
            ref = ops.axpy(state[f"B{l}.{w}"], env[f"B{l}.d{w}"], {"scalar": -1.0})
            assert np.array_equal(env[f"B{l}.{w}"], ref)


def test_training_chain_shape():
    spec = wl.mlp_train_chain(n_blocks=6)
    step = spec.nodes[spec.segments[1][0]:]
    # no staging COPY of X: the first GEMM reads the EXTERNAL X through its rebuilt tensor map
    assert len(step) == 3 * 6 + 2 + 9 * 6 + 2 * 5 + 2 * 6 == 96
    ops_ = {n.op for n in step}
    assert ops_ == {"GEMM_BF16", "GELU", "SUB", "SCALE_IMM", "TRANSPOSE", "GELU_BWD", "AXPY"}
    assert math.isclose(spec.nodes[spec.segments[1][0] + 19].attrs["scalar"], 2.0 / (128 * 768))
    staged = wl.mlp_train_chain(n_blocks=6, stage_x=True)
    assert len(staged.nodes) == len(spec.nodes) + 1 and staged.nodes[staged.segments[1][0]].op == "COPY"
