"""Seeded, counter-based synthetic value generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no chain op, no rebinding rule, no selector
cost); it only turns (seed, stream, index) into exactly-representable input values. Both sides
of every parity test draw their inputs from here (task rule ③: "only the seeded input generators
serve both, from a module of their own").

Recipe:
  h(seed, stream, i) = mix(mix(seed XOR mix(stream)) + i)      with mix = splitmix64 finaliser
  * fp32 uniform in [-1, 1):  k = h >> 40 (top 24 bits);  v = k * 2^-23 - 1   (exact in fp32)
  * bf16 uniform in [-1, 1):  k = h >> 56 (top 8 bits);   v = k / 128 - 1     (exact in bf16)
  * integer mode:             v = ((h >> 32) mod 5) - 2  in {-2..2}          (exact everywhere)
All arithmetic on the uint64 counters wraps mod 2^64.
"""
from __future__ import annotations

import numpy as np

U64 = np.uint64
_GOLDEN = U64(0x9E3779B97F4A7C15)
_M1 = U64(0xBF58476D1CE4E5B9)
_M2 = U64(0x94D049BB133111EB)

SEED = 0x19779  # SURVEY §8(d) C1 details: seed 0x19779


def _mix(z: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = np.asarray(z, dtype=U64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> U64(30))) * _M1
        z = (z ^ (z >> U64(27))) * _M2
    return z ^ (z >> U64(31))


def hash64(seed: int, stream: int, n: int, start: int = 0) -> np.ndarray:
    """h(seed, stream, i) for i in [start, start+n) as uint64."""
    s = _mix(np.array([stream & 0xFFFFFFFFFFFFFFFF], dtype=U64))
    base = _mix(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=U64) ^ s)
    idx = np.arange(start, start + n, dtype=U64)
    with np.errstate(over="ignore"):
        return _mix(base + idx)


def uniform_f32(seed: int, stream: int, n: int) -> np.ndarray:
    """fp32 values k*2^-23 - 1, k = top 24 bits of h. Exact in fp32, range [-1, 1)."""
    k = (hash64(seed, stream, n) >> U64(40)).astype(np.float64)
    return (k * 2.0**-23 - 1.0).astype(np.float32)


def int_f32(seed: int, stream: int, n: int) -> np.ndarray:
    """Integer-mode fp32 values in {-2,-1,0,1,2}."""
    k = ((hash64(seed, stream, n) >> U64(32)) % U64(5)).astype(np.int64) - 2
    return k.astype(np.float32)


def uniform_bf16_bits(seed: int, stream: int, n: int, scale_pow2: int = 0) -> np.ndarray:
    """bf16 values (k/128 - 1) * 2^scale_pow2 as uint16 bit patterns (exact in bf16)."""
    k = (hash64(seed, stream, n) >> U64(56)).astype(np.float64)
    v = ((k / 128.0 - 1.0) * 2.0**scale_pow2).astype(np.float32)
    return (v.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def int_bf16_bits(seed: int, stream: int, n: int) -> np.ndarray:
    """Integer-mode bf16 values in {-2..2} as uint16 bit patterns."""
    v = int_f32(seed, stream, n)
    return (v.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def gamma_bf16_bits(seed: int, stream: int, n: int) -> np.ndarray:
    """LayerNorm gains near 1: 1 + (j - 8)/128, j = (h >> 56) mod 16. Exact in bf16."""
    j = ((hash64(seed, stream, n) >> U64(56)) % U64(16)).astype(np.float64)
    v = (1.0 + (j - 8.0) / 128.0).astype(np.float32)
    return (v.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns to float32 (a bit shift, no rounding)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def stream_id(slot: int, replay: int) -> int:
    """Stream of external slot `slot` at replay `replay` ((slot<<20)|replay)."""
    return (slot << 20) | (replay & 0xFFFFF)


STATIC_REPLAY = 0xFFFFF  # replay index reserved for STATIC (weight) slots
