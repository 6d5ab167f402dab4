"""Alg. 1 LeanTile(), step by step in fp64.  TEST INFRASTRUCTURE ONLY.

    function LeanTile(tile_idx, iter_begin, iter_end)          §1
    O_acc = 0 (T_m x d);  m = -inf;  l = 0                      §8-9
    for iter = iter_begin to iter_end:                          §13 (half-open, reading C10)
        kk = iter * T_n                                         §14
        Q_f, K_f, V_f = LoadFragment(...)                       §16-18
        S_f = Q_f K_f^T            (scaled, reading C1)         §20
        m_new = max(m, rowmax(S_f))                             §21
        P_f = exp(S_f - m_new)                                  §22
        l_new = e^{m - m_new} l + rowsum(P_f)                   §23
        O_acc = P_f V_f + diag(e^{m - m_new}) O_acc             §24
        l = l_new, m = m_new                                    §25
    return O_acc, l, m                                          §27

Reading C5: a short last tile (N_k mod T_n != 0) holds only the valid rows.
Reading C13: §10-11's mm/nn (divisor/modulus 1) is indexing boilerplate -- one output tile
spans all of d and the T_m query rows are passed in directly.
"""
from __future__ import annotations

import numpy as np

from .rescale import PartialState, neutral


def lean_tile(q_rows: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float,
              iter_begin: int, iter_end: int, tile_n: int) -> PartialState:
    """Online softmax over LeanTile iterations [iter_begin, iter_end) of one output tile.

    q_rows (T_m, d); k, v (N_k, d) of ONE (batch, kv-head).  Returns the un-scaled
    (O_acc, m, l) -- NOT divided by l.
    """
    q_rows = np.atleast_2d(np.asarray(q_rows, dtype=np.float64))
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n_k = k.shape[0]
    c_n = -(-n_k // tile_n)
    if not (0 <= iter_begin < iter_end <= c_n):
        raise ValueError(f"bad iteration range [{iter_begin}, {iter_end}) for C_n={c_n}")
    st = neutral(q_rows.shape[0], q_rows.shape[1])           # §8-9
    o_acc, m, l = st.o, st.m, st.l
    for it in range(iter_begin, iter_end):                   # §13
        kk = it * tile_n                                     # §14
        k_f = k[kk:kk + tile_n]                              # §17 (short tail: C5)
        v_f = v[kk:kk + tile_n]                              # §18
        s_f = scale * (q_rows @ k_f.T)                       # §20
        m_new = np.maximum(m, s_f.max(axis=1))               # §21
        p_f = np.exp(s_f - m_new[:, None])                   # §22
        alpha = np.where(np.isfinite(m), np.exp(m - m_new), 0.0)   # e^{m - m_new}; m=-inf -> 0
        l_new = alpha * l + p_f.sum(axis=1)                  # §23
        o_acc = p_f @ v_f + alpha[:, None] * o_acc           # §24
        l, m = l_new, m_new                                  # §25
    return PartialState(o_acc, m, l)                         # §27
