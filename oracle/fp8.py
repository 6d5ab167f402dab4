"""OCP FP8 E4M3 codes -> fp64, for the FP8-KV inputs (NEXT-4).  TEST INFRASTRUCTURE ONLY.

Not in the paper (it streams 16-bit K/V); SURVEY.md §8(f) NEXT-4 adds an FP8 KV cache.
The attention the FP8 path computes is still Eq. 1, on the dequantised cache
K = code x k_scale, V = code x v_scale (per-tensor scales, reading C23); this
module only turns the stored bytes into their real values, from the format's definition:

    byte = s eeee mmm            (sign, 4 exponent bits with bias 7, 3 mantissa bits)
    e == 0:            (-1)^s * 2^(1-7) * (m / 8)           (subnormals, and +-0)
    0 < e, not NaN:    (-1)^s * 2^(e-7) * (1 + m / 8)
    e == 15, m == 7:   NaN                                   (the "fn" variant has no inf;
                                                              e == 15, m < 7 are normals,
                                                              so the largest is 448)
"""
from __future__ import annotations

import numpy as np


def e4m3_decode(codes) -> np.ndarray:
    """Real values (fp64) of an array of E4M3 bytes (any integer dtype, values 0..255)."""
    c = np.asarray(codes).astype(np.int64)
    if c.size and (c.min() < 0 or c.max() > 255):
        raise ValueError("E4M3 codes are bytes")
    s = (c >> 7) & 1
    e = (c >> 3) & 15
    m = c & 7
    mag = np.where(e == 0, np.ldexp(m / 8.0, -6), np.ldexp(1.0 + m / 8.0, e - 7))
    out = np.where(s == 1, -mag, mag)
    return np.where((e == 15) & (m == 7), np.nan, out)


def dequantize(codes, scale: float) -> np.ndarray:
    """The cache value of stored codes: code x scale (reading C23), fp64."""
    return e4m3_decode(codes) * float(scale)
