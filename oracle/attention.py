"""Eq. 1 of the paper, decode phase, in fp64 -- the parity reference.  TEST INFRASTRUCTURE ONLY.

P:89-92 (Eq. 1):  S = Q K^T,  P = softmax(S / sqrt(d)),  O = P V
P:105-107 (Table 1, decode column): Q K^T is 1 x d x N, softmax is 1 x N, P V is 1 x N x d.

Readings: C1 the scale (default 1/sqrt(d)) multiplies every score
before max/exp; C2 L = ln sum_j exp(s_j) (natural log, scaled-score domain), the logsumexp
Alg. 2 §39 writes; C3 q-head h_q reads KV head h_q // g (g = H_q / H_kv).

The softmax is evaluated as exp(s_j - max s) / sum exp(s_i - max s), which equals Eq. 1's
softmax exactly in real arithmetic (numerator and denominator share the factor e^{-max}).
S is materialised in full ("computing the large intermediate matrices").
"""
from __future__ import annotations

import numpy as np


def scores(q_row: np.ndarray, k: np.ndarray, scale: float) -> np.ndarray:
    """s_j = scale * sum_c q[c] k[j, c] for every key j (Eq. 1's S = Q K^T, scaled)."""
    q_row = np.asarray(q_row, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    return scale * (k @ q_row)


def decode_attention_unit(q_rows: np.ndarray, k: np.ndarray, v: np.ndarray, scale: float):
    """Decode attention for the q-heads ``q_rows`` (g, d) sharing one KV head k, v (n, d).

    Returns (O (g, d), L (g,)) in fp64.  P:89-92; L per Alg. 2 §39.
    """
    q_rows = np.atleast_2d(np.asarray(q_rows, dtype=np.float64))
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if k.ndim != 2 or v.shape != k.shape or q_rows.shape[1] != k.shape[1]:
        raise ValueError(f"shape mismatch q{q_rows.shape} k{k.shape} v{v.shape}")
    if k.shape[0] < 1:
        raise ValueError("empty context (DESIGN.md reading C6)")
    g, d = q_rows.shape
    O = np.empty((g, d), dtype=np.float64)
    L = np.empty((g,), dtype=np.float64)
    for i in range(g):
        s = scores(q_rows[i], k, scale)          # S row, 1 x N   (Table 1: 1 x d x N)
        m = s.max()
        p = np.exp(s - m)                        # softmax numerators, 1 x N
        l = p.sum()                              # softmax denominator (times e^{-m})
        O[i] = (p @ v) / l                       # O = P V        (Table 1: 1 x N x d)
        L[i] = m + np.log(l)                     # ln sum_j e^{s_j}
    return O, L


def decode_attention_multi(q: np.ndarray, k: np.ndarray, v: np.ndarray, ctx_lens, scale: float,
                           causal: bool = True, layout: str = "bhsd", block_table=None, page_size: int = 0):
    """N_q > 1 queries per request (NEXT-3; the paper's general N_q, Alg2§4 C_m):
    q (B, H_q, N_q, d).  Query i of request b is the cached token at position n_b - N_q + i;
    with ``causal`` it attends to keys [0, n_b - N_q + i] (the prefill-phase mask restricted
    to the new tokens), otherwise to all n_b keys.  Eq. 1 per query row.
    Returns O (B, H_q, N_q, d), L (B, H_q, N_q)."""
    q = np.asarray(q, dtype=np.float64)
    B, Hq, Nq, d = q.shape
    O = np.empty((B, Hq, Nq, d))
    L = np.empty((B, Hq, Nq))
    for i in range(Nq):
        lens_i = [int(n) - Nq + i + 1 if causal else int(n) for n in ctx_lens]
        o, l = _sliced(q[:, :, i], k, v, ctx_lens, lens_i, scale, layout, block_table, page_size)
        O[:, :, i], L[:, :, i] = o, l
    return O, L


def decode_attention_varq(q_rows: np.ndarray, k: np.ndarray, v: np.ndarray, ctx_lens, q_lens, scale: float,
                          causal: bool = True, layout: str = "bhsd", block_table=None, page_size: int = 0):
    """Heterogeneous batch (NEXT-3: decode mixed with speculative / chunked-prefill query
    blocks; the paper's general N_q per request): request b brings N_b =
    q_lens[b] query tokens.  q_rows holds, request after request, an (H_q, N_b, d) block:
    row (b, h_q, i) = sum_{b' < b} H_q N_b' + h_q N_b + i.  Query i of request b is the
    cached token n_b - N_b + i; with ``causal`` it attends to keys [0, n_b - N_b + i], else
    to all n_b keys.  Eq. 1 per row.  Returns O (rows, d), L (rows,)."""
    q_rows = np.asarray(q_rows, dtype=np.float64)
    Hkv = k.shape[0] if layout == "packed" else k.shape[1]
    d = q_rows.shape[-1]
    B = len(ctx_lens)
    Hq = q_rows.shape[0] // int(np.sum(q_lens))
    g = Hq // Hkv
    cu = np.concatenate([[0], np.cumsum(ctx_lens)]).astype(np.int64)
    O = np.empty((q_rows.shape[0], d))
    L = np.empty((q_rows.shape[0],))
    row = 0
    for b in range(B):
        n, nb = int(ctx_lens[b]), int(q_lens[b])
        for hq in range(Hq):
            h = hq // g
            if layout == "bhsd":
                kk, vv = k[b, h, :n], v[b, h, :n]
            elif layout == "packed":
                kk, vv = k[h, cu[b]:cu[b + 1]], v[h, cu[b]:cu[b + 1]]
            else:
                kk = paged_rows(k, block_table[b], h, n, page_size)
                vv = paged_rows(v, block_table[b], h, n, page_size)
            for i in range(nb):
                m = n - nb + i + 1 if causal else n
                o, l = decode_attention_unit(q_rows[row], kk[:m], vv[:m], scale)
                O[row], L[row] = o[0], l[0]
                row += 1
    return O, L


def _sliced(q, k, v, ctx_lens, lens_i, scale, layout, block_table, page_size):
    """decode_attention over the first lens_i[b] keys of every request."""
    B, Hq, d = q.shape
    Hkv = k.shape[0] if layout == "packed" else k.shape[1]
    g = Hq // Hkv
    cu = np.concatenate([[0], np.cumsum(ctx_lens)]).astype(np.int64)
    O = np.empty((B, Hq, d))
    L = np.empty((B, Hq))
    for b in range(B):
        n = int(ctx_lens[b])
        for h in range(Hkv):
            if layout == "bhsd":
                kk, vv = k[b, h, :n], v[b, h, :n]
            elif layout == "packed":
                kk, vv = k[h, cu[b]:cu[b + 1]], v[h, cu[b]:cu[b + 1]]
            else:
                kk = paged_rows(k, block_table[b], h, n, page_size)
                vv = paged_rows(v, block_table[b], h, n, page_size)
            m = lens_i[b]
            o, l = decode_attention_unit(q[b, h * g:(h + 1) * g], kk[:m], vv[:m], scale)
            O[b, h * g:(h + 1) * g] = o
            L[b, h * g:(h + 1) * g] = l
    return O, L


def paged_rows(pool: np.ndarray, block_table_row, h: int, n: int, page_size: int) -> np.ndarray:
    """The n context rows of KV head h of one request in a paged pool (num_pages, H_kv,
    page_size, d): token t is row t % page_size of page block_table_row[t // page_size]."""
    pages = [pool[int(block_table_row[i]), h] for i in range(-(-n // page_size))]
    return np.concatenate(pages, axis=0)[:n]


def decode_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, ctx_lens, scale: float,
                     layout: str = "bhsd", block_table=None, page_size: int = 0):
    """Batched decode attention.

    q: (B, H_q, d).  k, v: ``bhsd`` (B, H_kv, max_ctx, d) with request b valid for rows
    [0, ctx_lens[b]); or ``packed`` (H_kv, sum n_b, d), the paper's ragged layout
    with request b at rows cu_seqlens[b] .. cu_seqlens[b+1]; or ``paged`` pools
    (num_pages, H_kv, page_size, d) addressed through ``block_table`` [B][pages].
    Returns O (B, H_q, d) and L (B, H_q), fp64.
    """
    q = np.asarray(q, dtype=np.float64)
    B, Hq, d = q.shape
    Hkv = k.shape[0] if layout == "packed" else k.shape[1]
    if Hq % Hkv:
        raise ValueError("heads_q must be a multiple of heads_kv (reading C3)")
    g = Hq // Hkv
    cu = np.concatenate([[0], np.cumsum(ctx_lens)]).astype(np.int64)
    O = np.empty((B, Hq, d), dtype=np.float64)
    L = np.empty((B, Hq), dtype=np.float64)
    for b in range(B):
        n = int(ctx_lens[b])
        for h in range(Hkv):
            if layout == "bhsd":
                kk, vv = k[b, h, :n], v[b, h, :n]
            elif layout == "packed":
                kk, vv = k[h, cu[b]:cu[b + 1]], v[h, cu[b]:cu[b + 1]]
            elif layout == "paged":
                kk = paged_rows(k, block_table[b], h, n, page_size)
                vv = paged_rows(v, block_table[b], h, n, page_size)
            else:
                raise ValueError(layout)
            o, l = decode_attention_unit(q[b, h * g:(h + 1) * g], kk, vv, scale)
            O[b, h * g:(h + 1) * g] = o
            L[b, h * g:(h + 1) * g] = l
    return O, L
