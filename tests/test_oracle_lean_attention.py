"""Pins for oracle.lean_attention (Alg. 2 serial) and oracle.shard_combine.

Alg. 2 with any grid must reproduce Eq. 1 ("same exact attention output ...
regardless of the way the work might be split"); the sequence-shard combine must reproduce
the unsharded result (BASELINE.json north star; §4.1 associativity).
"""
import math

import numpy as np
import pytest

import oracle
import synth


def _random_problem(rng, layout):
    B = int(rng.integers(1, 4))
    Hkv = int(rng.integers(1, 4))
    g = int(rng.choice([1, 2, 4]))
    d = int(rng.choice([4, 8]))
    lens = [int(x) for x in rng.integers(1, 60, size=B)]
    maxn = max(lens)
    q = rng.normal(size=(B, Hkv * g, d)) * 2
    if layout == "bhsd":
        k = rng.normal(size=(B, Hkv, maxn, d))
        v = rng.normal(size=(B, Hkv, maxn, d))
    else:
        k = rng.normal(size=(Hkv, sum(lens), d))
        v = rng.normal(size=(Hkv, sum(lens), d))
    return q, k, v, lens, 1 / math.sqrt(d)


@pytest.mark.parametrize("layout", ["bhsd", "packed"])
@pytest.mark.parametrize("seed", range(6))
def test_alg2_equals_eq1_any_grid(layout, seed):
    rng = np.random.default_rng(seed)
    q, k, v, lens, scale = _random_problem(rng, layout)
    O_ref, L_ref = oracle.decode_attention(q, k, v, lens, scale, layout)
    for tile_n in (1, 4, 16):
        I = sum(-(-n // tile_n) for n in lens) * k.shape[1 if layout == "bhsd" else 0]
        for G in sorted({1, 2, 3, 5, I // 2 + 1, I, I + 3}):
            O, L = oracle.lean_attention(q, k, v, lens, scale, tile_n, G, layout)
            assert np.max(np.abs(O - O_ref)) <= 1e-12
            assert np.max(np.abs(L - L_ref)) <= 1e-12


def test_fig1_configuration_two_reductions():
    # Fig. 1 (2 heads, 5 tiles each, grid 5) -> exactly 2 tiles need a reduction
    rng = np.random.default_rng(7)
    d, tile_n = 4, 3
    q = rng.normal(size=(1, 2, d))
    k = rng.normal(size=(1, 2, 5 * tile_n, d))
    v = rng.normal(size=(1, 2, 5 * tile_n, d))
    O, L, st = oracle.lean_attention(q, k, v, [5 * tile_n], 0.5, tile_n, 5, return_stats=True)
    O_ref, L_ref = oracle.decode_attention(q, k, v, [5 * tile_n], 0.5)
    assert np.max(np.abs(O - O_ref)) <= 1e-12
    assert st["partials"] == 4 and st["folds"] == 4 and st["segments"] == 6


@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_shard_combine_equals_full(P):
    rng = np.random.default_rng(P)
    n, d, rows = 1000, 16, 3
    q = rng.normal(size=(rows, d)) * 2
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, d))
    O_ref, L_ref = oracle.decode_attention_unit(q, k, v, 0.25)
    o_parts, l_parts = [], []
    for r in range(P):
        a, b = (r * n) // P, ((r + 1) * n) // P
        o, l = oracle.decode_attention_unit(q, k[a:b], v[a:b], 0.25)
        o_parts.append(o)
        l_parts.append(l)
    O, L = oracle.combine_shards(np.stack(o_parts), np.stack(l_parts))
    assert np.max(np.abs(O - O_ref)) <= 1e-12 and np.max(np.abs(L - L_ref)) <= 1e-12
    # P = 1 is the identity
    O1, L1 = oracle.combine_shards(O_ref[None], L_ref[None])
    assert np.allclose(O1, O_ref, atol=1e-15) and np.allclose(L1, L_ref, atol=1e-15)


def test_synth_shards_tile_the_context():
    p = synth.Problem(2, 2, 2, 8, [37, 64], dtype="bf16", layout="bhsd")
    full = synth.fill_kv_cache(p, "k")
    for P in (2, 3):
        parts = [synth.fill_kv_cache(p, "k", token_range=synth.shard_bounds(p, r, P)) for r in range(P)]
        for b, n in enumerate(p.ctx_lens):
            rows = [parts[r][b, :, :synth.shard_bounds(p, r, P)[b][1] - synth.shard_bounds(p, r, P)[b][0]]
                    for r in range(P)]
            assert torch_equal(np_cat(rows), full[b, :, :n])


def np_cat(ts):
    import torch
    return torch.cat(ts, dim=1)


def torch_equal(a, b):
    import torch
    return torch.equal(a, b)
