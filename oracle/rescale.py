"""§4.1 "Softmax Re-scaling as Reduction", fp64.  TEST INFRASTRUCTURE ONLY.

P:274-280 -- the un-scaled partial of a KV block i of any length B_c^(i):
    S^(i) = Q K^(i)T,  m^(i) = rowmax S^(i),  l^(i) = rowsum e^{S^(i) - m^(i)},
    A^(i) = e^{S^(i) - m^(i)},  O~^(i) = A^(i) V^(i)
P:286-294 -- the softmax re-scaling operation f(x, y):
    m^(x,y) = max(m^(x), m^(y))
    l^(x,y) = e^{m^(x) - m^(x,y)} l^(x) + e^{m^(y) - m^(x,y)} l^(y)
    f(x,y)  = diag(e^{m^(x) - m^(x,y)}) O~^(x) + diag(e^{m^(y) - m^(x,y)}) O~^(y) = O~^(x,y)
    O^(x,y) = diag(l^(x,y))^{-1} f(x, y)
Alg. 2 §38-39 -- finalisation O = diag(l)^{-1} O, L = m + log(l).

Readings: C1 (scores carry the 1/sqrt(d) scale), C12 (fold un-scaled, normalise once at
the end).  The neutral element (O~ = 0, m = -inf, l = 0) is Alg. 1 §8-9's initial state
(P:371-372); e^{m_x - m_xy} with m_x = -inf is taken as exactly 0 (no -inf - -inf).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable

import numpy as np

from .attention import scores


@dataclass
class PartialState:
    """(O~ (rows, d), m (rows,), l (rows,)) -- P:276-280.  rows = T_m (query-tile rows)."""

    o: np.ndarray
    m: np.ndarray
    l: np.ndarray


def neutral(rows: int, d: int) -> PartialState:
    """Alg. 1 §8-9: O_acc = 0, m = -inf, l = 0."""
    return PartialState(np.zeros((rows, d)), np.full((rows,), -np.inf), np.zeros((rows,)))


def partial(q_rows: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float) -> PartialState:
    """Un-scaled partial of one KV block, materialised (no online update)."""
    q_rows = np.atleast_2d(np.asarray(q_rows, dtype=np.float64))
    g, d = q_rows.shape
    out = neutral(g, d)
    if k.shape[0] == 0:
        return out
    for i in range(g):
        s = scores(q_rows[i], k, scale)                 # S^(i)
        m = s.max()                                     # m^(i) = rowmax(S^(i))
        a = np.exp(s - m)                               # A^(i) = exp(S^(i) - m^(i))
        out.m[i] = m
        out.l[i] = a.sum()                              # l^(i) = rowsum(A^(i))
        out.o[i] = a @ np.asarray(v, dtype=np.float64)  # O~^(i) = A^(i) V^(i)
    return out


def _weight(m: np.ndarray, m_xy: np.ndarray) -> np.ndarray:
    """e^{m - m_xy}, with the neutral element's m = -inf giving exactly 0."""
    w = np.zeros_like(m)
    fin = np.isfinite(m)
    w[fin] = np.exp(m[fin] - m_xy[fin])
    return w


def combine(x: PartialState, y: PartialState) -> PartialState:
    """f(x, y) with its statistics."""
    if x.o.shape != y.o.shape:
        raise ValueError("shape mismatch")
    m_xy = np.maximum(x.m, y.m)                     # m^(x,y) = max(m^(x), m^(y))
    wx = _weight(x.m, m_xy)                         # e^{m^(x) - m^(x,y)}
    wy = _weight(y.m, m_xy)                         # e^{m^(y) - m^(x,y)}
    l_xy = wx * x.l + wy * y.l                      # l^(x,y)
    o_xy = wx[:, None] * x.o + wy[:, None] * y.o    # f(x,y) = O~^(x,y)
    return PartialState(o_xy, m_xy, l_xy)


def fold(states: Iterable[PartialState]) -> PartialState:
    """Left fold f(f(f(s0, s1), s2), ...) in the given order (Alg. 2 §27-36)."""
    it = iter(states)
    acc = next(it)
    for s in it:
        acc = combine(acc, s)
    return acc


def finalize(state: PartialState):
    """Alg. 2 §38-39: O = diag(l)^{-1} O, L = m + log(l)."""
    if np.any(state.l <= 0):
        raise ValueError("finalising the neutral element (l = 0)")
    return state.o / state.l[:, None], state.m + np.log(state.l)
