"""Host restatement of the ensemble's fixed-point moment arithmetic (test infrastructure).

A term v (already divided by the power of two 2^k nearest sigma) becomes M = trunc(|v| 2^64)
split into three 42-bit digits, negated for v < 0 (csrc/rk_sim.cu fx_digits); a moment is the
digit-wise int64 sum; its value is sum_i d_i 2^(42 i) / 2^64.  Python ints make the reference
sums exact."""
import math

import numpy as np

MASK = (1 << 42) - 1


def fx_scale(sigma2: float) -> float:
    return math.ldexp(1.0, math.floor(0.5 * math.log2(sigma2)))


def digits(v: float):
    m = int(abs(v) * 2.0 ** 64) if v != 0.0 else 0   # exact: a power-of-two rescale, then truncation
    d = [m & MASK, (m >> 42) & MASK, m >> 84]
    return [-x for x in d] if math.copysign(1.0, v) < 0 else d


def digits_array(vals):
    """(count, npix) float64 -> (3, npix) int64 digit sums over the count axis."""
    vals = np.asarray(vals, dtype=np.float64)
    out = np.zeros((3,) + vals.shape[1:], dtype=np.int64)
    flat = vals.reshape(vals.shape[0], -1)
    o = out.reshape(3, -1)
    for j in range(flat.shape[0]):
        for p in range(flat.shape[1]):
            d = digits(float(flat[j, p]))
            for q in range(3):
                o[q, p] += d[q]
    return out


def value(d0, d1, d2) -> int:
    return int(d0) + (int(d1) << 42) + (int(d2) << 84)


def moments(e, sigma2):
    """Accumulator (6, ...) of terms e (count, ...) as the library keeps it."""
    s = fx_scale(sigma2)
    v = np.asarray(e, dtype=np.float64) / s
    return np.concatenate([digits_array(v), digits_array(v * v)])
