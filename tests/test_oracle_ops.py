"""Pins for oracle/numerics.py and oracle/ops.py (no GPU).

Each check ties the oracle to something other than itself: IEEE-754 arithmetic done in Python
floats, ml_dtypes' bf16 conversion, closed forms, brute-force loops in exact integers, and the
SPEC worked example S:L122.
"""
import math
import struct

import ml_dtypes
import numpy as np
import pytest

from oracle import numerics as nm
from oracle import ops
from synth import splitmix as sm


def f32(x: float) -> float:
    """Round a Python float (binary64) to binary32 via the C library's conversion."""
    return struct.unpack("<f", struct.pack("<f", x))[0]


# ------------------------------------------------------------------ bf16 rounding

def test_bf16_matches_ml_dtypes_on_f32_inputs():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 3,
                        (rng.standard_normal(2000) * 1e-30).astype(np.float32),
                        (rng.integers(0, 2**16, 4000).astype(np.float32) / 2**8 + 1)])
    ref = x.astype(ml_dtypes.bfloat16).astype(np.float64)
    assert np.array_equal(nm.bf16_rne(x.astype(np.float64)), ref)


def test_bf16_ties_and_single_rounding():
    e = 2.0**-8
    assert nm.bf16_rne(np.array([1 + e]))[0] == 1.0               # tie -> even (down)
    assert nm.bf16_rne(np.array([1 + 3 * e]))[0] == 1 + 2.0**-6    # tie -> even (up)
    # direct f64->bf16 differs from f64->f32->bf16 here: a single rounding must go up
    x = 1 + e + 2.0**-30
    assert nm.bf16_rne(np.array([x]))[0] == 1 + 2.0**-7
    assert nm.bf16_rne(np.array([f32(x)]))[0] == 1.0
    assert np.isinf(nm.bf16_rne(np.array([3.5e38]))[0])
    assert nm.bf16_rne(np.array([-0.0]))[0] == 0.0


def test_bf16_bits_roundtrip():
    bits = np.arange(0, 2**16, 7, dtype=np.uint16)
    v = nm.bits_to_f64(bits)
    ok = np.isfinite(v)
    assert np.array_equal(nm.bf16_bits(v[ok]), bits[ok])


# ------------------------------------------------------------------ fp32 elementwise (a5)

def test_scale_worked_example():
    # ScaleByScalar(x=[2,4], s=3) -> [6,12]
    out = ops.scale_imm(np.array([2, 4], np.float32), {"scalar": 3.0})
    assert out.tolist() == [6.0, 12.0]


@pytest.mark.parametrize("op", ["add", "mul"])
def test_fp32_elementwise_is_ieee_single_rounding(op):
    a = sm.uniform_f32(sm.SEED, 11, 3000)
    b = sm.uniform_f32(sm.SEED, 12, 3000)
    a[:4] = [1e-30, 1.5, -2.5, 1.0]
    b[:4] = [1e-30, 2.0**-24, 7.0, 2.0**-24 * 3]
    got = getattr(ops, op)(a, b, {})
    for i in range(len(a)):
        x, y = float(a[i]), float(b[i])
        exact = x + y if op == "add" else x * y      # exact in binary64 for these operands
        assert got[i] == np.float32(f32(exact)), (i, x, y)


def test_window_touches_prefix_only():
    a = np.arange(10, dtype=np.float32)
    out = ops.add(a, a, {"n": 4})
    assert out.tolist() == [0, 2, 4, 6]


def test_reduce_sum_integer_exact_and_fsum():
    a = sm.int_f32(sm.SEED, 3, 256 * 16)
    out = ops.reduce_sum(a, {"cols": 256})
    for r in range(16):
        assert out[r] == sum(int(v) for v in a[r * 256:(r + 1) * 256])
    b = sm.uniform_f32(sm.SEED, 4, 256 * 8)
    out = ops.reduce_sum(b, {"cols": 256})
    for r in range(8):
        assert out[r] == np.float32(math.fsum(float(v) for v in b[r * 256:(r + 1) * 256]))


# ------------------------------------------------------------------ decoder nodes (a7)

def _ints(stream, n):
    return sm.int_f32(sm.SEED, stream, n).astype(np.float64)


@pytest.mark.parametrize("M,N,K", [(3, 5, 7), (16, 32, 64), (1, 16, 48)])
def test_gemm_bruteforce_integer_exact(M, N, K):
    a, w, b, r = _ints(1, M * K), _ints(2, N * K), _ints(3, N), _ints(4, M * N)
    got = ops.gemm_bf16(a, w, b, {"M": M, "N": N, "K": K, "bias": True}, residual=r)
    for i in range(M):
        for j in range(N):
            ref = sum(int(a[i * K + k]) * int(w[j * K + k]) for k in range(K)) + int(b[j]) + int(r[i * N + j])
            assert got[i * N + j] == ref     # |ref| <= 4K + 4 <= 260: exact in bf16 (8 bits)


def test_gemm_dropped_k_tile_is_caught():
    M, N, K = 8, 8, 128
    a = sm.uniform_f32(sm.SEED, 5, M * K).astype(np.float64)
    w = sm.uniform_f32(sm.SEED, 6, N * K).astype(np.float64)
    full = ops.gemm_bf16(a, w, None, {"M": M, "N": N, "K": K})
    a2 = a.reshape(M, K).copy()
    a2[:, 64:] = 0
    part = ops.gemm_bf16(a2.reshape(-1), w, None, {"M": M, "N": N, "K": K})
    rms = np.sqrt(np.mean(full ** 2))
    assert np.any(np.abs(part - full) > 2e-2 * np.abs(full) + 2e-2 * rms)


def test_gelu_closed_forms():
    assert ops.gelu_tanh(np.array([0.0]))[0] == 0.0
    assert abs(ops.gelu_tanh(np.array([1.0]))[0] - 0.8411919906082768) < 1e-15
    assert abs(ops.gelu_tanh(np.array([10.0]))[0] - 10.0) < 1e-12
    assert abs(ops.gelu_tanh(np.array([-10.0]))[0]) < 1e-12


def test_gemm_gelu_epilogue_order():
    a, w, b = np.array([1.0, 2.0]), np.array([0.5, -1.0]), np.array([0.25])
    got = ops.gemm_bf16(a, w, b, {"M": 1, "N": 1, "K": 2, "bias": True, "gelu": True})
    x = 0.5 - 2.0 + 0.25
    ref = 0.5 * x * (1 + math.tanh(math.sqrt(2 / math.pi) * (x + 0.044715 * x ** 3)))
    assert got[0] == nm.bf16_rne(np.array([ref]))[0]


def test_layernorm_closed_forms():
    cols = 8
    x = np.full(2 * cols, 0.75)
    g = nm.bits_to_f64(sm.gamma_bf16_bits(sm.SEED, 1, cols))
    b = nm.bits_to_f64(sm.uniform_bf16_bits(sm.SEED, 2, cols, -5))
    out = ops.layernorm(x, np.tile(g, 1), b, {"rows": 2, "cols": cols, "eps": 1e-5})
    assert np.array_equal(out, np.tile(b, 2))                       # constant row -> beta
    x = np.array([1.0, 3.0])
    out = ops.layernorm(x, np.array([1.0, 1.0]), np.array([0.0, 0.0]),
                        {"rows": 1, "cols": 2, "eps": 1e-5})
    s = 1 / math.sqrt(1 + 1e-5)                                      # mean 2, var 1
    assert out.tolist() == nm.bf16_rne(np.array([-s, s])).tolist()


def test_layernorm_bruteforce_rows():
    rows, cols = 3, 24
    x = nm.bits_to_f64(sm.uniform_bf16_bits(sm.SEED, 7, rows * cols))
    g = nm.bits_to_f64(sm.gamma_bf16_bits(sm.SEED, 8, cols))
    b = nm.bits_to_f64(sm.uniform_bf16_bits(sm.SEED, 9, cols, -5))
    out = ops.layernorm(x, g, b, {"rows": rows, "cols": cols, "eps": 1e-5})
    for r in range(rows):
        row = [float(v) for v in x[r * cols:(r + 1) * cols]]
        mu = math.fsum(row) / cols
        var = math.fsum((v - mu) ** 2 for v in row) / cols
        for c in range(cols):
            ref = (row[c] - mu) / math.sqrt(var + 1e-5) * g[c] + b[c]
            assert abs(out[r * cols + c] - ref) <= abs(ref) * 2.0**-8 + 1e-12


def test_attention_uniform_when_logits_equal():
    T, H, D = 6, 2, 4
    qkv = np.zeros((T, 3, H, D))
    v = _ints(10, T * H * D).reshape(T, H, D)
    qkv[:, 2] = v
    out = ops.attn_causal(qkv.reshape(-1), {"T": T, "H": H, "D": D, "scale": 0.125}).reshape(T, H, D)
    for i in range(T):
        ref = v[:i + 1].mean(axis=0)                     # causal: uniform over j <= i
        assert np.array_equal(out[i], nm.bf16_rne(ref))


def test_attention_bruteforce():
    T, H, D = 5, 2, 3
    qkv = sm.uniform_f32(sm.SEED, 13, T * 3 * H * D).astype(np.float64)
    out = ops.attn_causal(qkv, {"T": T, "H": H, "D": D, "scale": 0.125}).reshape(T, H, D)
    X = qkv.reshape(T, 3, H, D)
    for h in range(H):
        for i in range(T):
            s = [0.125 * sum(X[i, 0, h, d] * X[j, 1, h, d] for d in range(D)) for j in range(i + 1)]
            m = max(s)
            e = [math.exp(v - m) for v in s]
            z = math.fsum(e)
            for d in range(D):
                ref = math.fsum(e[j] / z * X[j, 2, h, d] for j in range(i + 1))
                assert abs(out[i, h, d] - ref) <= abs(ref) * 2.0**-8 + 1e-12


def test_allreduce_integer_partials():
    parts = [_ints(20 + r, 64) for r in range(4)]
    out = ops.allreduce_sum(parts)
    assert np.array_equal(out, parts[0] + parts[1] + parts[2] + parts[3])


def test_scale_t_is_scale_imm_with_a_device_scalar():
    # S:L122 worked example through the CGCT scalar-as-tensor form
    out = ops.scale_t(np.array([2, 4], np.float32), np.array([3.0], np.float32), {})
    assert out.tolist() == [6.0, 12.0]
    a = sm.uniform_f32(sm.SEED, 30, 1000)
    assert np.array_equal(ops.scale_t(a, np.array([0.75], np.float32), {}),
                          ops.scale_imm(a, {"scalar": 0.75}))


def test_c3_fused_residual_matches_unfused_within_bf16():
    """residual adds may be fused into the GEMM epilogue. The fused chain (7 nodes per
    layer) keeps the same seeded weights (same slot indices) and differs from the 9-node chain only
    by the intermediate bf16 rounding of the GEMM output before the add: a few bf16 ulps."""
    from oracle.chain import eval_chain
    from synth import workloads as wl
    f = wl.c3_chain(T=8, n_layers=2, fuse_residual=True)
    u = wl.c3_chain(T=8, n_layers=2)
    assert len(f.nodes) == 14 and len(u.nodes) == 18
    ef = eval_chain(f, wl.external_values(f, 0), wl.static_values(f))
    eu = eval_chain(u, wl.external_values(u, 0), wl.static_values(u))
    a, b = ef["L1.h2"], eu["L1.h2"]
    assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-2
    assert not np.array_equal(a, b)          # the fusion does change the rounding
