"""Pins for oracle.attention (Eq. 1) against things other than itself.

* mpmath brute force at 50 digits on tiny inputs (independent arithmetic);
* SPEC worked values;
* closed forms: q = 0 -> O = mean V, L = ln n; census input -> exact integers;
  a single dominant key -> O = its value row;
* invariants: row-stochasticity, score-shift (through K), key permutation, GQA grouping,
  layout independence.
"""
import math

import mpmath
import numpy as np
import pytest

import oracle

mpmath.mp.dps = 50


def _mp_attention(q, k, v, scale):
    """Eq. 1 with mpmath at 50 digits, written from the definition softmax(x)_j = e^x_j / sum e^x."""
    n, d = k.shape
    s = [mpmath.mpf(scale) * mpmath.fsum(mpmath.mpf(q[c]) * mpmath.mpf(k[j, c]) for c in range(d))
         for j in range(n)]
    e = [mpmath.e ** sj for sj in s]
    z = mpmath.fsum(e)
    o = [mpmath.fsum(e[j] * mpmath.mpf(v[j, c]) for j in range(n)) / z for c in range(d)]
    return np.array([float(x) for x in o]), float(mpmath.log(z))


@pytest.mark.parametrize("seed", range(12))
def test_brute_force_mpmath(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 65))
    d = int(rng.integers(1, 9))
    q = rng.normal(size=d) * rng.uniform(0.1, 4)
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, d))
    scale = 1 / math.sqrt(d) if seed % 2 else float(rng.uniform(0.2, 3))
    O, L = oracle.decode_attention_unit(q[None], k, v, scale)
    O_mp, L_mp = _mp_attention(q, k, v, scale)
    assert np.max(np.abs(O[0] - O_mp)) <= 1e-13 * max(1.0, np.max(np.abs(O_mp)))
    assert abs(L[0] - L_mp) <= 1e-13 * max(1.0, abs(L_mp))


def test_spec_examples():
    # N_q=1, N_k=1, d=2, Q=[1,0], K=[[1,0]], V=[[5,7]], scale=1 -> O=[5,7], L=1
    O, L = oracle.decode_attention_unit(np.array([[1.0, 0.0]]), np.array([[1.0, 0.0]]),
                                        np.array([[5.0, 7.0]]), 1.0)
    assert np.array_equal(O[0], [5.0, 7.0]) and L[0] == 1.0
    # Q=[0], K=[[3],[9]], V=[[1],[2]] -> O=[1.5], L=log 2
    O, L = oracle.decode_attention_unit(np.array([[0.0]]), np.array([[3.0], [9.0]]),
                                        np.array([[1.0], [2.0]]), 0.7)
    assert O[0, 0] == 1.5 and L[0] == pytest.approx(math.log(2), abs=1e-15)


def test_zero_query_is_mean_and_log_n():
    rng = np.random.default_rng(5)
    for n in (1, 7, 128, 1000):
        v = rng.normal(size=(n, 16))
        O, L = oracle.decode_attention_unit(np.zeros((1, 16)), rng.normal(size=(n, 16)), v, 0.25)
        assert np.allclose(O[0], v.mean(axis=0), rtol=0, atol=1e-14)
        assert L[0] == pytest.approx(math.log(n), abs=1e-14)


def test_dominant_key():
    rng = np.random.default_rng(6)
    n, d = 300, 8
    k = rng.normal(size=(n, d)) * 0.01
    q = np.ones(d)
    k[123] = 100.0                       # score 800 above every other one
    v = rng.normal(size=(n, d))
    O, L = oracle.decode_attention_unit(q[None], k, v, 1.0)
    assert np.allclose(O[0], v[123], atol=1e-12)
    assert L[0] == pytest.approx(800.0, abs=1e-9)


def test_census_closed_form():
    # DESIGN.md D3: q = 0, V[t, c] = C [c == (t // T_c) mod d] -> O_c = C #{t: (t//T_c)%d == c} / n
    n, d, tc = 4096, 64, 256
    C = n // tc
    t = np.arange(n)
    v = np.zeros((n, d))
    v[t, (t // tc) % d] = C
    O, L = oracle.decode_attention_unit(np.zeros((1, d)), np.ones((n, d)), v, 0.125)
    expect = np.array([C * np.sum((t // tc) % d == c) / n for c in range(d)])
    assert np.array_equal(O[0], expect)
    assert set(np.unique(O[0])) <= {0.0, 1.0}
    assert L[0] == pytest.approx(math.log(n), abs=1e-13)


@pytest.mark.parametrize("seed", range(4))
def test_row_stochastic_shift_and_permutation(seed):
    rng = np.random.default_rng(100 + seed)
    n, d = 257, 32
    q = rng.normal(size=d) * 2
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, d))
    scale = 1 / math.sqrt(d)
    O, L = oracle.decode_attention_unit(q[None], k, v, scale)
    # S:61 row-stochasticity: sum_j exp(s_j - L) = 1
    s = scale * np.einsum("jc,c->j", k, q)
    assert abs(np.exp(s - L[0]).sum() - 1.0) <= 1e-12
    # S:62 shift invariance, realised through K: k_j += w with scale q.w = c for all j
    c = 3.75
    w = q * (c / (scale * (q @ q)))
    O2, L2 = oracle.decode_attention_unit(q[None], k + w[None, :], v, scale)
    assert np.max(np.abs(O2 - O)) <= 1e-12
    assert L2[0] - L[0] == pytest.approx(c, abs=1e-12)
    # S:63 permutation equivariance over the N_k axis
    perm = rng.permutation(n)
    O3, L3 = oracle.decode_attention_unit(q[None], k[perm], v[perm], scale)
    assert np.max(np.abs(O3 - O)) <= 1e-12 and abs(L3[0] - L[0]) <= 1e-12


def test_gqa_grouping_and_layouts():
    # Reading C3: q-head h reads KV head h // g.  Give every KV head a constant V row so the
    # output of each q-head names the KV head it attended to.
    rng = np.random.default_rng(7)
    B, Hkv, g, d = 2, 3, 4, 8
    lens = [5, 11]
    maxn = max(lens)
    k = rng.normal(size=(B, Hkv, maxn, d))
    v = np.zeros((B, Hkv, maxn, d))
    for b in range(B):
        for h in range(Hkv):
            v[b, h, :, :] = 10 * b + h
    q = rng.normal(size=(B, Hkv * g, d))
    O, L = oracle.decode_attention(q, k, v, lens, 0.3)
    for b in range(B):
        for hq in range(Hkv * g):
            assert np.allclose(O[b, hq], 10 * b + hq // g, atol=1e-12)
    # packed layout gives the same numbers
    kp = np.concatenate([k[b, :, :lens[b]] for b in range(B)], axis=1)
    vp = np.concatenate([v[b, :, :lens[b]] for b in range(B)], axis=1)
    O2, L2 = oracle.decode_attention(q, kp, vp, lens, 0.3, layout="packed")
    assert np.array_equal(O, O2) and np.array_equal(L, L2)
    # padding rows beyond n_b are never read
    k[0, :, lens[0]:] = np.nan
    O3, _ = oracle.decode_attention(q, k, v, lens, 0.3)
    assert np.array_equal(O, O3)


def test_errors():
    with pytest.raises(ValueError):
        oracle.decode_attention_unit(np.zeros((1, 4)), np.zeros((3, 5)), np.zeros((3, 5)), 1.0)
    with pytest.raises(ValueError):
        oracle.decode_attention_unit(np.zeros((1, 4)), np.zeros((0, 4)), np.zeros((0, 4)), 1.0)


def test_paged_layout_is_the_same_rows():
    # NEXT-4 paged pools: the oracle's gather through the block table reproduces the BHSD
    # result bit for bit (the layouts hold the same bf16 rows)
    import synth
    for ps in (16, 64):
        base = dict(batch=3, heads_q=4, heads_kv=2, head_dim=32, ctx_lens=[100, 17, 64], dtype="bf16",
                    dist="D2", seed=9)
        pb = synth.Problem(**base)
        pp = synth.Problem(**base, layout="paged", page_size=ps)
        q = synth.to_f64(synth.gen_q(pb))
        O1, L1 = oracle.decode_attention(q, synth.to_f64(synth.fill_kv_cache(pb, "k")),
                                         synth.to_f64(synth.fill_kv_cache(pb, "v")), pb.ctx_lens, pb.scale)
        bt, npages = synth.paged_meta(pp)
        assert sorted(set(bt[0, :-(-100 // ps)].tolist()) | set(bt[1, :2].tolist())) is not None
        kp = synth.fill_kv_cache(pp, "k")
        assert kp.shape == (npages, 2, ps, 32)
        O2, L2 = oracle.decode_attention(q, synth.to_f64(kp), synth.to_f64(synth.fill_kv_cache(pp, "v")),
                                         pp.ctx_lens, pp.scale, "paged", block_table=bt, page_size=ps)
        assert np.array_equal(O1, O2) and np.array_equal(L1, L2)
        # pages of one request are scattered, and no page is shared between requests
        used = [bt[b, i] for b, n in enumerate(pp.ctx_lens) for i in range(-(-n // ps))]
        assert len(set(used)) == len(used)


def test_multi_query_causal_against_mpmath_and_truncation():
    # NEXT-3 (N_q > 1): query i is the cached token n - N_q + i; causally it sees keys
    # [0, n - N_q + i].  Pinned against mpmath with the mask written out, and against
    # single-query attention over the truncated cache.
    rng = np.random.default_rng(21)
    B, Hkv, g, Nq, d = 2, 2, 2, 3, 6
    lens = [9, 5]
    k = rng.normal(size=(B, Hkv, 9, d))
    v = rng.normal(size=(B, Hkv, 9, d))
    q = rng.normal(size=(B, Hkv * g, Nq, d))
    O, L = oracle.decode_attention_multi(q, k, v, lens, 0.4, causal=True)
    for b in range(B):
        for hq in range(Hkv * g):
            for i in range(Nq):
                m = lens[b] - Nq + i + 1
                o_mp, l_mp = _mp_attention(q[b, hq, i], k[b, hq // g, :m], v[b, hq // g, :m], 0.4)
                assert np.max(np.abs(O[b, hq, i] - o_mp)) <= 1e-13 and abs(L[b, hq, i] - l_mp) <= 1e-13
    On, Ln = oracle.decode_attention_multi(q, k, v, lens, 0.4, causal=False)
    for i in range(Nq):
        Oi, Li = oracle.decode_attention(q[:, :, i], k, v, lens, 0.4)
        assert np.array_equal(On[:, :, i], Oi) and np.array_equal(Ln[:, :, i], Li)
    # the last query of a causal block sees the whole cache
    Ol, Ll = oracle.decode_attention(q[:, :, Nq - 1], k, v, lens, 0.4)
    assert np.max(np.abs(O[:, :, Nq - 1] - Ol)) <= 1e-13


def test_heterogeneous_batch_against_mpmath():
    # NEXT-3 heterogeneous batches: request b brings N_b queries (rows (b, h_q, i) in
    # per-request (H_q, N_b) blocks); query i sees keys [0, n_b - N_b + i] when causal.
    # Pinned against mpmath with the row layout and the mask written out independently.
    rng = np.random.default_rng(22)
    Hkv, g, d = 2, 3, 5
    lens, qls = [7, 4, 9], [1, 4, 2]
    Hq = Hkv * g
    k = rng.normal(size=(3, Hkv, 9, d))
    v = rng.normal(size=(3, Hkv, 9, d))
    rows = sum(Hq * n for n in qls)
    q = rng.normal(size=(rows, d))
    for causal in (True, False):
        O, L = oracle.decode_attention_varq(q, k, v, lens, qls, 0.7, causal=causal)
        assert O.shape == (rows, d) and L.shape == (rows,)
        r = 0
        for b in range(3):
            for hq in range(Hq):
                for i in range(qls[b]):
                    m = lens[b] - qls[b] + i + 1 if causal else lens[b]
                    o_mp, l_mp = _mp_attention(q[r], k[b, hq // g, :m], v[b, hq // g, :m], 0.7)
                    assert np.max(np.abs(O[r] - o_mp)) <= 1e-13 and abs(L[r] - l_mp) <= 1e-13
                    r += 1
