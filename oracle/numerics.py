"""bf16 rounding for the oracle (SURVEY §8(c) O1 and ambiguity 11: "bf16 RNE everywhere").

bf16_rne rounds a float64 value ONCE to the nearest bfloat16 (ties to even); there is no
intermediate float32 step, so it is the plain definition "round the exact value to bf16".
Pinned in tests against ml_dtypes.bfloat16 on float32 inputs (where float32->bf16 is itself a
single rounding) and against hand-built tie cases.
"""
from __future__ import annotations

import numpy as np

BF16_MAX = (2.0 - 2.0**-7) * 2.0**127
_MIN_NORMAL = 2.0**-126


def bf16_rne(x) -> np.ndarray:
    """Round float64 values to the nearest bf16 value (RNE); returns float64 holding bf16 values."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                               # x = m * 2^e, 0.5 <= |m| < 1
    r = np.ldexp(np.rint(np.ldexp(m, 8)), e - 8)     # keep 8 significant bits, ties-to-even
    small = np.abs(x) < _MIN_NORMAL                  # subnormal range: fixed quantum 2^-133
    if np.any(small):
        r = np.where(small, np.ldexp(np.rint(np.ldexp(x, 133)), -133), r)
    # overflow: values at or beyond max + half an ulp (2^120) round to infinity
    over = np.abs(x) >= BF16_MAX + 2.0**119
    if np.any(over):
        r = np.where(over, np.copysign(np.inf, x), r)
    return r


def bf16_bits(v) -> np.ndarray:
    """bf16-representable float64 values -> uint16 bit patterns (exact: a truncating shift)."""
    f = np.asarray(v, dtype=np.float64).astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bits_to_f64(bits) -> np.ndarray:
    """uint16 bf16 bit patterns -> exact float64 values."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    with np.errstate(invalid="ignore"):
        return b.view(np.float32).astype(np.float64)
