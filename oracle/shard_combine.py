"""Sequence-shard combine of normalised partials (O_r, L_r).  TEST INFRASTRUCTURE ONLY.

BASELINE.json north star: each GPU r runs decode attention on a contiguous slice of every
head's context and emits its normalised output O_r and logsumexp L_r; after an all-gather
the final output is the softmax re-scaling reduction (§4.1) of the per-rank
partials, which is exact for any split by associativity.

In normalised form a partial (O~_r, m_r, l_r) is (O_r = O~_r / l_r, L_r = m_r + ln l_r).
Folding all P partials with f and finalising gives
    L = ln sum_r e^{L_r},     O = sum_r e^{L_r - L} O_r
which is what this function computes, with the max subtracted for range (reading C12).
"""
from __future__ import annotations

import numpy as np


def combine_shards(o_parts: np.ndarray, lse_parts: np.ndarray):
    """o_parts (P, rows, d), lse_parts (P, rows) -> O (rows, d), L (rows,), fp64."""
    o_parts = np.asarray(o_parts, dtype=np.float64)
    lse_parts = np.asarray(lse_parts, dtype=np.float64)
    m = lse_parts.max(axis=0)                          # max_r L_r
    w = np.exp(lse_parts - m[None, :])                 # e^{L_r - max}
    s = w.sum(axis=0)
    L = m + np.log(s)                                  # ln sum_r e^{L_r}
    O = (w[:, :, None] * o_parts).sum(axis=0) / s[:, None]   # sum_r e^{L_r - L} O_r
    return O, L
