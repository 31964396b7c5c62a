"""O1 — per-node definitions of the chain ops (SPEC opcode algebra).

Representation: f32 slots are numpy float32 arrays; bf16 slots are float64 arrays holding exact
bf16 values. Every function is the plain mathematical definition followed by ONE rounding to the
slot's storage type:
  * fp32 elementwise ops are numpy float32 arithmetic (IEEE-754 binary32, round-to-nearest-even,
    one rounding per op, no fused multiply-add) — SURVEY §8(a) a5 "rounded to nearest once".
  * REDUCE_SUM accumulates in float64 and rounds once to fp32 (O1).
  * bf16 ops compute in float64 and round once to bf16 (O1, ambiguity 11).
"""
from __future__ import annotations

import math

import numpy as np

from .numerics import bf16_rne


def _n(a, attrs):
    return int(attrs.get("n", a.shape[0]))


# ------------------------------------------------------------------ elementwise (a5)

def add(a, b, attrs, dtype="f32"):
    """ADD(a,b)[i] = a[i] + b[i] over the first n elements."""
    n = _n(a, attrs)
    if dtype == "f32":
        return np.add(a[:n], b[:n], dtype=np.float32)
    return bf16_rne(a[:n].astype(np.float64) + b[:n].astype(np.float64))


def mul(a, b, attrs, dtype="f32"):
    """MUL(a,b)[i] = a[i] * b[i]."""
    n = _n(a, attrs)
    if dtype == "f32":
        return np.multiply(a[:n], b[:n], dtype=np.float32)
    return bf16_rne(a[:n].astype(np.float64) * b[:n].astype(np.float64))


def scale_imm(a, attrs, dtype="f32"):
    """SCALE_IMM(a,c)[i] = a[i] * c, c a by-value float (S:L122 worked example [2,4]*3=[6,12])."""
    n = _n(a, attrs)
    c = attrs["scalar"]
    if dtype == "f32":
        return np.multiply(a[:n], np.float32(c), dtype=np.float32)
    return bf16_rne(a[:n].astype(np.float64) * float(np.float32(c)))


def scale_t(a, s, attrs, dtype="f32"):
    """SCALE_T(a, s)[i] = a[i] * s[0]: the CGCT rewrite of a by-value scalar into a 1-element
    device tensor ("alters the type of parameter as a GPU-resident tensor")."""
    n = _n(a, attrs)
    return np.multiply(a[:n], np.float32(s[0]), dtype=np.float32)


def copy(a, attrs, dtype="f32"):
    """COPY(a)[i] = a[i]."""
    return a[:_n(a, attrs)].copy()


# ------------------------------------------------------------------ training-shaped chain (NEXT-4)

def sub(a, b, attrs, dtype="bf16"):
    """SUB(a,b)[i] = a[i] - b[i], one rounding (bf16)."""
    n = _n(a, attrs)
    return bf16_rne(a[:n].astype(np.float64) - b[:n].astype(np.float64))


def axpy(a, b, attrs, dtype="bf16"):
    """AXPY(a,b)[i] = a[i] + c * b[i], c = attrs['scalar'] as fp32 (the SGD step W - lr * dW with
    c = -lr), one rounding (bf16)."""
    n = _n(a, attrs)
    c = float(np.float32(attrs["scalar"]))
    return bf16_rne(a[:n].astype(np.float64) + c * b[:n].astype(np.float64))


def gelu_grad(x):
    """d/dx of the tanh-approximate GELU 0.5 x (1 + tanh(u)), u = k0 (x + k1 x^3):
    0.5 (1 + tanh u) + 0.5 x (1 - tanh^2 u) k0 (1 + 3 k1 x^2)."""
    k0, k1 = math.sqrt(2.0 / math.pi), 0.044715
    t = np.tanh(k0 * (x + k1 * x ** 3))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * k0 * (1.0 + 3.0 * k1 * x * x)


def gelu(a, attrs, dtype="bf16"):
    """GELU(a)[i] (tanh approximation), one rounding (bf16)."""
    n = _n(a, attrs)
    return bf16_rne(gelu_tanh(a[:n].astype(np.float64)))


def gelu_bwd(dy, x, attrs, dtype="bf16"):
    """GELU_BWD(dy, x)[i] = dy[i] * GELU'(x[i]) (chain rule through the activation), one rounding."""
    n = _n(dy, attrs)
    return bf16_rne(dy[:n].astype(np.float64) * gelu_grad(x[:n].astype(np.float64)))


def transpose(a, attrs, dtype="bf16"):
    """TRANSPOSE: out[c, r] = in[r, c] for in = [n / cols, cols] row-major (exact copy)."""
    n, cols = _n(a, attrs), int(attrs["cols"])
    return a[:n].reshape(n // cols, cols).T.reshape(-1).copy()


def reduce_sum(a, attrs, dtype="f32"):
    """REDUCE_SUM(a)[r] = sum_c a[r, c] over rows of `cols`, f64 accumulate, one fp32 rounding
    (SURVEY §8(a) a6, §8(c) O1)."""
    n = _n(a, attrs)
    cols = int(attrs.get("cols", 256))
    rows = a[:n].astype(np.float64).reshape(n // cols, cols)
    return rows.sum(axis=1).astype(np.float32)


# ------------------------------------------------------------------ decoder nodes (a7)

def layernorm(x, g, b, attrs):
    """LN over rows: (x - mean) / sqrt(var + eps) * g + b, population variance, f64, one bf16
    rounding (SURVEY §8(c) O1 'LAYERNORM'; eps 1e-5 per ambiguity 11)."""
    rows, cols, eps = int(attrs["rows"]), int(attrs["cols"]), float(attrs["eps"])
    X = x.astype(np.float64).reshape(rows, cols)
    mean = X.mean(axis=1, keepdims=True)
    var = ((X - mean) ** 2).mean(axis=1, keepdims=True)
    Y = (X - mean) / np.sqrt(var + eps) * g.astype(np.float64) + b.astype(np.float64)
    return bf16_rne(Y).reshape(-1)


def gelu_tanh(x):
    """tanh-approximate GELU: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))) (ambiguity 11)."""
    x = np.asarray(x, dtype=np.float64)
    return 0.5 * x * (1.0 + np.tanh(math.sqrt(2.0 / math.pi) * (x + 0.044715 * x ** 3)))


def gemm_bf16(a, w, bias, attrs, residual=None):
    """o[i,j] = bf16( epi( sum_k a[i,k] w[j,k] + bias[j] ) ) with epi = GELU if attrs['gelu'],
    then + residual[i,j] if given; the whole epilogue in f64 before ONE rounding (O1 'GEMM_BF16').
    a: [M,K], w: [N,K] (nn.Linear layout), bias: [N]."""
    M, N, K = int(attrs["M"]), int(attrs["N"]), int(attrs["K"])
    A = a.astype(np.float64).reshape(M, K)
    W = w.astype(np.float64).reshape(N, K)
    acc = A @ W.T
    if attrs.get("bias", False):
        acc = acc + bias.astype(np.float64).reshape(1, N)
    if attrs.get("gelu", False):
        acc = gelu_tanh(acc)
    if residual is not None:
        acc = acc + residual.astype(np.float64).reshape(M, N)
    return bf16_rne(acc).reshape(-1)


def attn_causal(qkv, attrs):
    """Per head h: softmax(Q_h K_h^T * scale + mask) V_h with mask[i,j] = -inf for j > i, f64,
    one bf16 rounding (O1 'ATTN_CAUSAL'; scale 0.125 = 1/sqrt(64), ambiguity 11).
    qkv: [T, 3*H*D] with column blocks q | k | v, each head-major ([H, D])."""
    T, H, D, scale = int(attrs["T"]), int(attrs["H"]), int(attrs["D"]), float(attrs["scale"])
    X = qkv.astype(np.float64).reshape(T, 3, H, D)
    out = np.empty((T, H, D))
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    for h in range(H):
        q, k, v = X[:, 0, h, :], X[:, 1, h, :], X[:, 2, h, :]
        s = (q @ k.T) * scale
        s[mask] = -np.inf
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        p = p / p.sum(axis=1, keepdims=True)
        out[:, h, :] = p @ v
    return bf16_rne(out).reshape(-1)


def allreduce_sum(partials):
    """ALLREDUCE_SUM: out = sum over ranks of the partials, in f64, one bf16 rounding
    (O1 'ALLREDUCE_SUM'; P:L66 'collective operations' under TP)."""
    acc = np.zeros_like(np.asarray(partials[0], dtype=np.float64))
    for p in partials:
        acc = acc + np.asarray(p, dtype=np.float64)
    return bf16_rne(acc)
