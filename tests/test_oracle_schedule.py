"""Pins for oracle.schedule (§4.3 / Eq. 2 / Alg. 2 §4-18, §26, §41).

* the paper's Fig. 1 schedule (golden, P:42 + P:261 + P:412);
* Eq. 2 arithmetic and the remainder rule (golden);
* the literal Alg. 2 §26 formula drops a contributor on Fig. 1 (reading C9);
* Alg. 2's per-CTA walk == brute-force owner enumeration, exhaustively on small cases;
* structural invariants (coverage, balance <= 1, unique host, <= 1 partial per CTA, peers
  contiguous, non-host = first segment, non-finishing host = last segment);
* FA2 / FlashDecoding recovery and fixed-split quantization efficiency.
"""
import itertools
import os

import numpy as np

import pytest

import oracle
from oracle.schedule import Segment

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line)
    return rows


def test_fig1_golden():
    rows = [tuple(int(x) for x in r.split()) for r in _read_rows("fig1_schedule.txt")]
    segs = oracle.stream_k_segments([5, 5], 5)
    assert [s.row() for s in segs] == rows
    # SM0 and SM1 get 2 LeanTiles of h0, SM2 gets 1
    h0 = {s.cta: s.end - s.begin for s in segs if s.unit == 0}
    assert h0 == {0: 2, 1: 2, 2: 1}


def _expand(rle):
    out = []
    for tok in rle.split():
        n, v = tok.split("x")
        out += [int(v)] * int(n)
    return out


def test_eq2_golden():
    for row in _read_rows("eq2_arithmetic.txt"):
        lhs, rhs = row.split("->")
        kind, *args = lhs.split()
        expect = _expand(rhs)
        if kind == "eq2":
            B, H, N, T, G = map(int, args)
            c_n = [-(-N // T)] * (B * H)
        elif kind == "ragged":
            lens = [int(x) for x in args[0].split(",")]
            h, T, G = int(args[1]), int(args[2]), int(args[3])
            c_n = [-(-n // T) for _ in range(h) for n in lens]   # heads -> total context
        else:
            I, G = int(args[0]), int(args[1])
            c_n = [I]
        counts = oracle.iters_per_cta(sum(c_n), G)
        assert counts == expect, row
        segs = oracle.stream_k_segments(c_n, G)
        per = [0] * G
        for s in segs:
            per[s.cta] += s.end - s.begin
        assert per == expect
    assert sum(oracle.iters_per_cta(1728, 216)) == 1728
    assert oracle.quantization_efficiency(oracle.stream_k_segments([10], 4), 4) == pytest.approx(10 / 12)


def test_literal_alg2_line26_drops_a_contributor():
    # Alg. 2 §26 literally: last_cta = tile_iter_end / C_n.  On Fig. 1, head 0's host (CTA 0)
    # would wait only on CTA 1 and miss CTA 2's partial (reading C9).
    segs = oracle.stream_k_segments([5, 5], 5)
    assert oracle.last_cta_literal(5, 0) == 1 and oracle.last_cta_literal(5, 1) == 2
    true_last = {s.unit: s.last_cta for s in segs}
    assert true_last == {0: 2, 1: 4}
    contributors = {u: sorted({s.cta for s in segs if s.unit == u}) for u in (0, 1)}
    assert contributors == {0: [0, 1, 2], 1: [2, 3, 4]}


def _check_invariants(c_n, G, segs):
    I = sum(c_n)
    off = [0]
    for c in c_n:
        off.append(off[-1] + c)
    # coverage / disjointness of global iterations
    seen = []
    for s in segs:
        seen += list(range(off[s.unit] + s.begin, off[s.unit] + s.end))
    assert sorted(seen) == list(range(I))
    # balance <= 1
    per = [0] * G
    for s in segs:
        per[s.cta] += s.end - s.begin
    assert max(per) - min(per) <= 1
    by_cta = {}
    for s in segs:
        by_cta.setdefault(s.cta, []).append(s)
    for u in range(len(c_n)):
        us = sorted([s for s in segs if s.unit == u], key=lambda s: s.begin)
        hosts = [s for s in us if s.host]
        assert len(hosts) == 1 and hosts[0].begin == 0            # unique host, owns iter 0
        h = hosts[0]
        ctas = [s.cta for s in us]
        assert ctas == list(range(h.cta, h.cta + len(us)))          # contiguous peers
        assert ctas[-1] == h.last_cta
        assert (len(us) == 1) == h.finishing
        for s in us[1:]:
            assert by_cta[s.cta][0] == s                            # non-host = first segment
        if not h.finishing:
            assert by_cta[h.cta][-1] == h                           # waiting host = last segment
    for g, ss in by_cta.items():
        assert sum(1 for s in ss if not s.host) <= 1                # <= 1 partial per CTA


def test_walk_equals_owner_enumeration_exhaustive():
    n_cases = 0
    for n_units in range(1, 5):
        for c_n in itertools.product(range(1, 7), repeat=n_units):
            I = sum(c_n)
            for G in range(1, I + 1):
                a = oracle.stream_k_segments(list(c_n), G)
                b = oracle.segments_from_owner_table(list(c_n), G)
                assert a == b, (c_n, G)
                _check_invariants(c_n, G, a)
                n_cases += 1
    assert n_cases > 20000


def test_owner_closed_form_and_idle_ctas():
    for I in range(1, 60):
        for G in range(1, 70):
            table = oracle.owner_table(I, G)
            assert [oracle.owner(I, G, i) for i in range(I)] == table
            segs = oracle.stream_k_segments([I], G)
            assert len({s.cta for s in segs}) == min(I, G)          # G > I: idle CTAs


def test_fa2_and_flashdecoding_recovery():
    # grid == #output tiles -> FA2 (one full tile per CTA)
    c_n = [7, 7, 7, 7]
    segs = oracle.stream_k_segments(c_n, 4)
    assert [(s.cta, s.unit, s.begin, s.end, s.host, s.finishing) for s in segs] == \
           [(u, u, 0, 7, True, True) for u in range(4)]
    # grid == s * #tiles with s | C_n -> FlashDecoding's equal split
    c_n = [6, 6, 6]
    segs = oracle.stream_k_segments(c_n, 6)
    assert [(s.unit, s.begin, s.end) for s in segs] == \
           [(0, 0, 3), (0, 3, 6), (1, 0, 3), (1, 3, 6), (2, 0, 3), (2, 3, 6)]
    fs = oracle.fixed_split_segments(c_n, 6, 2)
    assert sorted((s.unit, s.begin, s.end) for s in fs) == sorted((s.unit, s.begin, s.end) for s in segs)


def test_fixed_split_efficiency():
    # S:232 / S:258: 56 tiles, grid 108, split 1 -> 56/108
    fs = oracle.fixed_split_segments([4] * 56, 108, 1)
    load = [0] * 108
    for s in fs:
        load[s.cta] += s.end - s.begin
    assert sum(1 for x in load if x == 0) == 52
    assert oracle.quantization_efficiency(fs, 108) == pytest.approx(56 / 108)
    # 2 tiles of C_n=5, split 2 -> chunks 3 + 2
    fs = oracle.fixed_split_segments([5, 5], 4, 2)
    assert [(s.unit, s.end - s.begin) for s in fs] == [(0, 3), (0, 2), (1, 3), (1, 2)]
    # stream-K is never less efficient than fixed-split
    for c_n, G, s in [([5, 5], 4, 2), ([9] * 7, 16, 2), ([3, 17, 8], 5, 3)]:
        assert oracle.quantization_efficiency(oracle.stream_k_segments(c_n, G), G) >= \
            oracle.quantization_efficiency(oracle.fixed_split_segments(c_n, G, s), G)


def test_segments_from_ranges_generalises_alg2():
    rng = np.random.default_rng(3)
    for trial in range(300):
        c_n = [int(x) for x in rng.integers(1, 9, size=int(rng.integers(1, 6)))]
        I = sum(c_n)
        # equal ranges reproduce stream_k_segments exactly
        G = int(rng.integers(1, I + 3))
        begins = [oracle.cta_range(I, G, g)[0] for g in range(G)] + [I]
        assert oracle.segments_from_ranges(c_n, begins) == oracle.stream_k_segments(c_n, G)
        # random contiguous ranges == brute force over the per-iteration owner table
        cuts = sorted(set(int(x) for x in rng.integers(1, I, size=int(rng.integers(0, I)))) if I > 1 else set())
        begins = [0] + list(cuts) + [I]
        segs = oracle.segments_from_ranges(c_n, begins)
        own = []
        for v in range(len(begins) - 1):
            own += [v] * (begins[v + 1] - begins[v])
        off = np.concatenate([[0], np.cumsum(c_n)])
        brute = []
        for u in range(len(c_n)):
            first, last = off[u], off[u + 1] - 1
            start = first
            for it in range(first, last + 1):
                if it == last or own[it + 1] != own[it]:
                    brute.append(Segment(own[it], u, int(start - first), int(it + 1 - first), start == first,
                                         it == last, own[last]))
                    start = it + 1
        assert sorted(segs, key=lambda s: (s.cta, s.unit)) == sorted(brute, key=lambda s: (s.cta, s.unit))


def test_balanced_ranges_properties():
    """The dynamic schedule's layout (oracle.balanced_ranges): each Eq. 2 range (reading C8)
    is its head followed by k equal chunks; the pieces tile [0, I) in order; claims are every
    head in range order, then chunk j of every range, j = 0, 1, ..."""
    for I, G, hp, mc in [(65536, 148, 940, 2), (32768, 148, 940, 2), (245056, 148, 940, 2), (10, 4, 500, 1),
                         (7, 10, 940, 2), (1000, 1, 900, 3), (149, 148, 500, 1), (5000, 37, 800, 4)]:
        begins, claim = oracle.balanced_ranges(I, G, hp, mc)
        sizes = np.diff(begins)
        assert begins[0] == 0 and begins[-1] == I and np.all(sizes >= 1)
        assert sorted(claim) == list(range(len(begins) - 1))
        bset = set(begins)
        heads = []
        for g in range(G):
            lo, hi = oracle.cta_range(I, G, g)
            if lo == hi:
                continue
            assert lo in bset and hi in bset                    # every Eq. 2 range is a union of pieces
            inner = [x for x in begins if lo <= x <= hi]
            pieces = np.diff(inner)
            L = hi - lo
            t0 = L * (1000 - hp) // 1000
            s = max(mc, -(-t0 // 8))
            k = len(pieces) - 1
            assert k == min(t0 // s, (L - 1) // s) and k <= 8   # k chunks of s, head >= 1
            assert np.all(pieces[1:] == s) and pieces[0] == L - k * s
            heads.append(begins.index(lo))
        assert claim[:len(heads)] == heads                      # heads first, in range order
        rest = claim[len(heads):]
        rounds = [begins[v + 1] - begins[v] for v in rest]
        assert all(r >= 1 for r in rounds)
    # head share 1000: no tail -- exactly Alg. 2's equal ranges, claimed in order
    for I, G in [(65536, 148), (10, 4), (7, 10)]:
        begins, claim = oracle.balanced_ranges(I, G, 1000, 2)
        exp = sorted({oracle.cta_range(I, G, g)[0] for g in range(G)} | {I})
        assert begins == exp and claim == list(range(len(begins) - 1))
    # hand example: I = 10, G = 4 (ranges 3, 3, 2, 2), half tails of 1 LeanTile
    assert oracle.balanced_ranges(10, 4, 500, 1) == ([0, 2, 3, 5, 6, 7, 8, 9, 10], [0, 2, 4, 6, 1, 3, 5, 7])


def test_alg2_with_virtual_ctas_equals_eq1():
    rng = np.random.default_rng(4)
    q = rng.normal(size=(2, 3, 8)) * 2
    lens = [300, 77]
    k = rng.normal(size=(2, 3, 300, 8))
    v = rng.normal(size=(2, 3, 300, 8))
    O_ref, L_ref = oracle.decode_attention(q, k, v, lens, 0.35)
    c_n = [-(-n // 16) for n in lens for _ in range(3)]
    for G in (1, 3, 7, 40):
        begins, _ = oracle.balanced_ranges(sum(c_n), G, 700, 1)
        O, L = oracle.lean_attention(q, k, v, lens, 0.35, 16, G, begins=begins)
        assert np.max(np.abs(O - O_ref)) <= 1e-12 and np.max(np.abs(L - L_ref)) <= 1e-12


def test_weighted_ranges_properties_and_hand_values():
    """oracle.weighted_ranges (SM-rate-weighted Eq. 2): pinned by hand values,
    brute force and the properties the formula fixes."""
    # hand values: I = 10, w = (1, 2, 2): R = 7, begins = (0, 1 + 7/5, 2 + 21/5, 3 + 7) floored
    assert oracle.weighted_ranges(10, [1, 2, 2]) == [0, 2, 6, 10]
    assert oracle.weighted_ranges(7, [3, 1]) == [0, 4, 7]          # 1 + floor(5 * 3 / 4) = 4
    assert oracle.weighted_ranges(3, [1, 1, 1, 1, 1]) == [0, 1, 2, 3, 3, 3]   # I < G: trailing CTAs idle
    assert oracle.weighted_ranges(5, [1 << 20, 1]) == [0, 3, 5]    # 1 + floor(3 * 2^20 / (2^20 + 1)); the tiny weight keeps 2
    rng = np.random.default_rng(7)
    for trial in range(300):
        G = int(rng.integers(1, 200))
        I = int(rng.integers(0, 300000))
        w = [int(x) for x in rng.integers(1, 1 << 20, size=G)]
        if trial % 3 == 0:
            w = [int(x) for x in rng.integers(60000, 70000, size=G)]   # calibrated weights: +-8%
        b = oracle.weighted_ranges(I, w)
        W, R = sum(w), max(I - G, 0)
        sizes = np.diff(b)
        assert b[0] == 0 and b[-1] == I and np.all(sizes[:min(I, G)] >= 1) and np.all(sizes[min(I, G):] == 0)
        # each range within one LeanTile of 1 + its exact share R w_g / W (brute force, fractions)
        from fractions import Fraction
        for g in range(0, min(I, G), max(1, G // 20)):
            assert abs(Fraction(int(sizes[g])) - 1 - Fraction(R * w[g], W)) < 1
    # equal weights: sizes differ by at most one and sum to I (Eq. 2's balance, reading C8's
    # multiset of sizes, though the longer ranges are spread rather than first)
    for I, G in [(65536, 148), (32768, 148), (245056, 148), (10, 4), (7, 10), (149, 148)]:
        sizes = np.diff(oracle.weighted_ranges(I, [5] * G))
        assert sizes.sum() == I and sizes.max() - sizes.min() <= 1
        assert sorted(sizes.tolist()) == sorted(oracle.iters_per_cta(I, G))
    # scale invariance: multiplying every weight by c changes nothing
    assert oracle.weighted_ranges(12345, [3, 7, 11]) == oracle.weighted_ranges(12345, [300, 700, 1100])


def test_alg2_over_weighted_ranges_equals_eq1():
    rng = np.random.default_rng(5)
    q = rng.normal(size=(2, 4, 8)) * 2
    lens = [333, 91]
    k = rng.normal(size=(2, 2, 333, 8))
    v = rng.normal(size=(2, 2, 333, 8))
    O_ref, L_ref = oracle.decode_attention(q, k, v, lens, 0.4)
    c_n = [-(-n // 16) for n in lens for _ in range(2)]
    for G in (1, 2, 5, 13, 60):
        w = [int(x) for x in rng.integers(1, 1000, size=G)]
        begins = oracle.weighted_ranges(sum(c_n), w)
        O, L = oracle.lean_attention(q, k, v, lens, 0.4, 16, G, begins=begins)
        assert np.max(np.abs(O - O_ref)) <= 1e-12 and np.max(np.abs(L - L_ref)) <= 1e-12


def test_fixed_split_ranges_match_fixed_split_segments():
    # the range form of FD's split == the chunk list of fixed_split_segments
    for c_n, s in [([5, 5], 2), ([7, 3, 9], 3), ([1, 2, 3], 4), ([16] * 5, 4)]:
        begins = oracle.fixed_split_ranges(c_n, s)
        segs = oracle.segments_from_ranges(c_n, begins)
        ref = oracle.fixed_split_segments(c_n, 10 ** 6, s)
        assert [(x.unit, x.begin, x.end, x.host, x.finishing) for x in segs] == \
               [(x.unit, x.begin, x.end, x.host, x.finishing) for x in ref]
    # the split heuristic: pinned by exact values below (test_fa2_num_splits_hand_derived)


@pytest.mark.parametrize("units,max_cn,sms,expect", [
    # FlashAttention-2's num_splits heuristic (FlashDecoding's split rule, the paper's FD
    # baseline P:505; "FD opts not to split ... [when] the total number of heads in the batch
    # exceeds the number of SMs"), evaluated BY HAND.  With w(s) = units*s/sms waves,
    # eff(s) = w / ceil(w); no split if units >= 0.8*sms; else the smallest s <= min(128, sms,
    # max_cn) with eff(s) >= 0.85 * max_s eff(s).
    (1, 10 ** 6, 108, 92),   # eff(s) = s/108, max 1 at s = 108; 0.85*108 = 91.8 -> s = 92
    (56, 2, 108, 1),         # s <= 2: eff(1) = 56/108 = .5185, eff(2) = 1.037/2 = .5185 -> 1
    (56, 2048, 108, 5),      # eff 1:.519 2:.519 3:.778 4:.691 5:2.593/3=.864 >= .85 (max 1 at s=27)
    (56, 2048, 148, 5),      # eff 1:.378 2:.757 3:.568 4:.757 5:1.892/2=.946 >= .85 (max 1 at s=37)
    (32, 2048, 148, 4),      # c2: eff 1:.216 2:.432 3:.649 4:.865 >= .85 (max 1 at s=37)
    (64, 512, 148, 2),       # c3 units: eff 1:.432 2:.865 >= .85 (max 1 at s=37)
    (10, 3, 148, 3),         # max_cn caps s at 3: eff(3) = .203 is the max -> 3
    (118, 4, 148, 1),        # 118 < 118.4: every eff(s) = .797 = max -> s = 1
    (119, 4, 148, 1),        # 119 >= 0.8 * 148: no split at all
    (200, 64, 148, 1),
    (128, 2048, 148, 1),     # batch 4 x 32 heads fills 80% of 148 SMs
])
def test_fa2_num_splits_hand_derived(units, max_cn, sms, expect):
    assert oracle.fa2_num_splits(units, max_cn, sms) == expect
