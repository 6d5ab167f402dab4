"""Alg. 2 "Lean Attention" executed serially in fp64.  TEST INFRASTRUCTURE ONLY.

Runs every CTA's segments (Alg. 1 LeanTile per segment, §16), the non-host branch
(StorePartials into Op[g], mp[g], lp[g] + Signal, §19-23) and the host branch (wait on
flags[g+1 .. last_cta] and fold with the re-scaling operator in ascending CTA order,
§24-36; finalise, §38-39).  The CTAs' concurrency is replaced by two phases (all LeanTile
calls, then all host folds) -- the same dataflow, since a host only ever reads partials of
higher-indexed CTAs that were published at the end of their first segment.

Used to pin that the stream-K decomposition + fixup reproduces Eq. 1 ("same exact
attention output ... regardless of the way the work might be split").
"""
from __future__ import annotations

import numpy as np

from .leantile import lean_tile
from .rescale import combine, finalize
from .schedule import segments_from_ranges, stream_k_segments


def unit_order(batch: int, heads_kv: int, layout: str):
    """Linearisation order of work units (b, h_kv): P:412 (bhsd: batch -> heads) and
    P:432 (packed ragged: heads -> total context); reading C14."""
    if layout == "bhsd":
        return [(b, h) for b in range(batch) for h in range(heads_kv)]
    if layout == "packed":
        return [(b, h) for h in range(heads_kv) for b in range(batch)]
    raise ValueError(layout)


def lean_attention(q, k, v, ctx_lens, scale: float, tile_n: int, grid: int,
                   layout: str = "bhsd", return_stats: bool = False, begins=None):
    """Alg. 2 on (B, H_q, d) queries and a bhsd / packed KV cache; returns O, L (fp64).
    ``begins`` replaces §9's equal ranges by explicit per-CTA range boundaries (the
    virtual CTAs of the dynamic schedule); ``grid`` is then ignored."""
    q = np.asarray(q, dtype=np.float64)
    B, Hq, d = q.shape
    Hkv = k.shape[1] if layout == "bhsd" else k.shape[0]
    g_sz = Hq // Hkv
    cu = np.concatenate([[0], np.cumsum(ctx_lens)]).astype(np.int64)
    units = unit_order(B, Hkv, layout)

    def kv(u):
        b, h = units[u]
        n = int(ctx_lens[b])
        if layout == "bhsd":
            return k[b, h, :n], v[b, h, :n]
        return k[h, cu[b]:cu[b + 1]], v[h, cu[b]:cu[b + 1]]

    c_n = [-(-int(ctx_lens[b]) // tile_n) for (b, _h) in units]
    segs = stream_k_segments(c_n, grid) if begins is None else segments_from_ranges(c_n, begins)

    partials = {}     # Op[g], mp[g], lp[g]  (§20-22) -- written at most once per CTA
    hosts = []
    for s in segs:                                              # §10-16
        b, h = units[s.unit]
        kk, vv = kv(s.unit)
        st = lean_tile(q[b, h * g_sz:(h + 1) * g_sz], kk, vv, scale, s.begin, s.end, tile_n)
        if not s.host:                                          # §19-23
            if s.cta in partials:
                raise AssertionError(f"CTA {s.cta} would store a second partial")
            partials[s.cta] = st
        else:
            hosts.append((s, st))

    O = np.full((B, Hq, d), np.nan)
    L = np.full((B, Hq), np.nan)
    folds = 0
    for s, st in hosts:
        if not s.finishing:                                     # §24-25
            for cta in range(s.cta + 1, s.last_cta + 1):        # §27 (reading C9)
                st = combine(st, partials[cta])                 # §28-35 (reading C11)
                folds += 1
        o, l = finalize(st)                                     # §38-39
        b, h = units[s.unit]
        O[b, h * g_sz:(h + 1) * g_sz] = o
        L[b, h * g_sz:(h + 1) * g_sz] = l
    if return_stats:
        return O, L, {"segments": len(segs), "partials": len(partials), "folds": folds}
    return O, L
