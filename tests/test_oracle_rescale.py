"""Pins for oracle.rescale (§4.1) and oracle.leantile (Alg. 1).

* SPEC worked values for combine / finalize / lean_tile;
* identity law, bitwise;
* associativity: every permutation x every bracketing of k <= 5 partials agrees within
  1e-12 (BASELINE.json) -- and equals the MATERIALISED partial of the union of the blocks
  (the closed form of §4.1), so a wrong sign/exponent in f fails;
* split-point invariance vs Eq. 1;
* LeanTile over any range == the materialised partial of that token range; full range
  finalised == Eq. 1; tile-size independence; monotone running max.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle.rescale import PartialState


def _st(o, m, l):
    return PartialState(np.array([o], dtype=float), np.array([m], dtype=float),
                        np.array([l], dtype=float))


def test_spec_combine_values():
    # x=(O~=[2], m=1, l=1), y=(O~=[3], m=0, l=1) -> (2 + 3/e, 1, 1 + 1/e)
    r = oracle.combine(_st([2.0], 1.0, 1.0), _st([3.0], 0.0, 1.0))
    assert r.o[0, 0] == pytest.approx(2 + 3 / math.e, abs=1e-15)
    assert r.m[0] == 1.0 and r.l[0] == pytest.approx(1 + 1 / math.e, abs=1e-15)
    assert r.o[0, 0] == pytest.approx(3.10364, abs=1e-5) and r.l[0] == pytest.approx(1.36788, abs=1e-5)
    # equal maxima -> plain addition
    r = oracle.combine(_st([4.0], 2.0, 3.0), _st([4.0], 2.0, 3.0))
    assert (r.o[0, 0], r.m[0], r.l[0]) == (8.0, 2.0, 6.0)


def test_identity_bitwise():
    rng = np.random.default_rng(0)
    s = PartialState(rng.normal(size=(3, 5)), rng.normal(size=3) * 30, rng.uniform(0.5, 9, size=3))
    for r in (oracle.combine(oracle.neutral(3, 5), s), oracle.combine(s, oracle.neutral(3, 5))):
        assert np.array_equal(r.o, s.o) and np.array_equal(r.m, s.m) and np.array_equal(r.l, s.l)


def test_finalize_values():
    # S:115-116
    O, L = oracle.finalize(_st([5.0, 7.0], 1.0, 1.0))
    assert np.array_equal(O[0], [5.0, 7.0]) and L[0] == 1.0
    O, L = oracle.finalize(_st([2.0, 4.0], 0.0, 2.0))
    assert np.array_equal(O[0], [1.0, 2.0]) and L[0] == pytest.approx(math.log(2), abs=1e-16)
    with pytest.raises(ValueError):
        oracle.finalize(oracle.neutral(1, 2))


def _bracketings(items):
    """Every full binary bracketing of the sequence ``items`` (Catalan many)."""
    if len(items) == 1:
        yield items[0]
        return
    for i in range(1, len(items)):
        for left in _bracketings(items[:i]):
            for right in _bracketings(items[i:]):
                yield oracle.combine(left, right)


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_associativity_all_orders_and_groupings(k):
    rng = np.random.default_rng(10 + k)
    d = 6
    q = rng.normal(size=(1, d))
    worst = 0.0
    for trial in range(3):
        lens = rng.integers(1, 9, size=k)
        blocks = []
        for n in lens:
            # m spread +-50: scores shifted per block through a K component along q
            kk = rng.normal(size=(n, d)) + (rng.uniform(-50, 50) / (q @ q.T))[0, 0] * q
            blocks.append((kk, rng.normal(size=(n, d))))
        parts = [oracle.partial(q, kk, vv, 1.0) for kk, vv in blocks]
        union = oracle.partial(q, np.concatenate([b[0] for b in blocks]),
                               np.concatenate([b[1] for b in blocks]), 1.0)
        O_ref, L_ref = oracle.finalize(union)
        for perm in itertools.permutations(range(k)):
            for r in _bracketings([parts[i] for i in perm]):
                O, L = oracle.finalize(r)
                err = np.max(np.abs(O - O_ref)) / np.max(np.abs(O_ref))
                worst = max(worst, err, abs(L[0] - L_ref[0]) / abs(L_ref[0]))
                # l^((x,y),z) = l^(x,y,z) relative to the common max
                assert abs(r.m[0] - union.m[0]) <= 1e-13 * abs(union.m[0])
                assert abs(r.l[0] - union.l[0]) <= 1e-12 * union.l[0]
    assert worst <= 1e-12


@pytest.mark.parametrize("seed", range(3))
def test_split_point_invariance(seed):
    rng = np.random.default_rng(20 + seed)
    n, d = 97, 16
    q = rng.normal(size=(2, d)) * 2
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, d))
    O_ref, L_ref = oracle.decode_attention_unit(q, k, v, 0.25)
    for c in range(1, n):
        x = oracle.partial(q, k[:c], v[:c], 0.25)
        y = oracle.partial(q, k[c:], v[c:], 0.25)
        O, L = oracle.finalize(oracle.combine(x, y))
        assert np.max(np.abs(O - O_ref)) <= 1e-12 and np.max(np.abs(L - L_ref)) <= 1e-12


def test_lean_tile_spec_example():
    # one iteration, T_n=1, scale=1, q=[1,0], k=[[1,0]], v=[[5,7]] -> ([5,7], 1, 1)
    st = oracle.lean_tile(np.array([[1.0, 0.0]]), np.array([[1.0, 0.0]]),
                          np.array([[5.0, 7.0]]), 1.0, 0, 1, 1)
    assert np.array_equal(st.o[0], [5.0, 7.0]) and st.m[0] == 1.0 and st.l[0] == 1.0


@pytest.mark.parametrize("tile_n", [1, 2, 3, 16, 64, 1000])
def test_lean_tile_ranges_match_materialised_partial(tile_n):
    rng = np.random.default_rng(tile_n)
    n, d = 203, 12
    q = rng.normal(size=(3, d)) * 2
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, d))
    c_n = -(-n // tile_n)
    O_ref, L_ref = oracle.decode_attention_unit(q, k, v, 0.3)
    st = oracle.lean_tile(q, k, v, 0.3, 0, c_n, tile_n)
    O, L = oracle.finalize(st)
    assert np.max(np.abs(O - O_ref)) <= 1e-12 and np.max(np.abs(L - L_ref)) <= 1e-12
    for a, b in [(0, 1), (c_n - 1, c_n), (c_n // 3, max(c_n // 3 + 1, 2 * c_n // 3))]:
        if not 0 <= a < b <= c_n:
            continue
        st = oracle.lean_tile(q, k, v, 0.3, a, b, tile_n)
        ref = oracle.partial(q, k[a * tile_n:b * tile_n], v[a * tile_n:b * tile_n], 0.3)
        assert np.max(np.abs(st.m - ref.m)) <= 1e-13 * np.max(np.abs(ref.m))
        assert np.max(np.abs(st.l - ref.l) / ref.l) <= 1e-13
        assert np.max(np.abs(st.o - ref.o)) <= 1e-12 * np.max(np.abs(ref.o))


def test_lean_tile_monotone_max_and_errors():
    rng = np.random.default_rng(3)
    q = rng.normal(size=(1, 4))
    k = rng.normal(size=(40, 4))
    v = rng.normal(size=(40, 4))
    prev = -np.inf
    for e in range(1, 11):
        st = oracle.lean_tile(q, k, v, 1.0, 0, e, 4)
        assert st.m[0] >= prev and st.l[0] > 0
        prev = st.m[0]
    with pytest.raises(ValueError):
        oracle.lean_tile(q, k, v, 1.0, 3, 3, 4)
    with pytest.raises(ValueError):
        oracle.lean_tile(q, k, v, 1.0, 0, 11, 4)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_fold_every_order_equals_the_materialised_union(k):
    """oracle.fold is Alg. 2's host loop (§27-36): a left fold f(f(f(s0, s1), s2) ..).
    In EVERY order of k <= 5 block partials (m spread +-50) it must equal the materialised
    partial of the union of the blocks (§4.1's closed form) -- a dropped weight,
    a wrong sign in an exponent or an unscaled l fails this; finalising it gives Eq. 1."""
    rng = np.random.default_rng(40 + k)
    d = 5
    q = rng.normal(size=(2, d))
    for trial in range(3):
        lens = rng.integers(1, 8, size=k)
        blocks = []
        for n in lens:
            kk = rng.normal(size=(n, d)) + rng.uniform(-50, 50) * q[0] / (q[0] @ q[0])
            blocks.append((kk, rng.normal(size=(n, d))))
        parts = [oracle.partial(q, kk, vv, 1.0) for kk, vv in blocks]
        K = np.concatenate([b[0] for b in blocks])
        V = np.concatenate([b[1] for b in blocks])
        union = oracle.partial(q, K, V, 1.0)
        O_ref, L_ref = oracle.decode_attention_unit(q, K, V, 1.0)
        for perm in itertools.permutations(range(k)):
            r = oracle.fold(parts[i] for i in perm)
            assert np.max(np.abs(r.m - union.m)) <= 1e-13 * np.max(np.abs(union.m))
            assert np.max(np.abs(r.l - union.l) / union.l) <= 1e-12
            assert np.max(np.abs(r.o - union.o)) <= 1e-12 * np.max(np.abs(union.o))
            O, L = oracle.finalize(r)
            assert np.max(np.abs(O - O_ref)) <= 1e-12 and np.max(np.abs(L - L_ref)) <= 1e-12
    # the neutral element anywhere in the sequence changes nothing, bitwise (Alg1§8-9)
    a = oracle.fold([parts[0], oracle.neutral(2, d)] + parts[1:])
    b = oracle.fold(parts)
    assert np.array_equal(a.o, b.o) and np.array_equal(a.m, b.m) and np.array_equal(a.l, b.l)
