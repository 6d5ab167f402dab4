"""la_plan_update (per-step re-planning, P:430-432 Lean Ragged Batching) and the host-side
invariants of the schedules the kernel relies on -- host-only plans, no GPU needed.

* An update must produce exactly the schedule a fresh plan with the same launch grid
  produces (bit-exact: the export rows), for every schedule and layout.
* The dynamic schedule's fold-tree counters (DecodeArgs::grp_count) must be distinct per
  (unit, group) within one launch: ADVICE r01 found shapes where a CTA ends one unit's
  group and hosts the next unit's first group on the same counter.
* la_plan_info.quantization_efficiency equals the oracle's definition on the
  oracle's own enumeration of the same schedule.
"""
import numpy as np
import pytest

import oracle
import synth
from oracle.lean_attention import unit_order


@pytest.fixture(scope="module")
def la():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as pkg
    pkg.lib()
    return pkg


def _lens(rng, batch, lo=1, hi=20000):
    return [int(x) for x in rng.integers(lo, hi, size=batch)]


@pytest.mark.parametrize("schedule", ["streamk", "dynamic", "fixed_split", "sequential"])
@pytest.mark.parametrize("layout", ["bhsd", "packed", "paged"])
def test_update_equals_fresh_plan(la, schedule, layout):
    rng = np.random.default_rng(21)
    for trial in range(12):
        batch = int(rng.integers(1, 7))
        hkv = int(rng.integers(1, 9))
        g = int(rng.choice([1, 2, 4, 8]))
        tile = int(rng.choice([32, 64, 128]))
        cap = 20000
        lens0 = _lens(rng, batch, hi=cap)
        kw = dict(tile_n=tile, host_only=True, schedule=schedule, layout=layout, engine="mma")
        if layout == "bhsd":
            kw["max_ctx"] = cap
        if layout == "paged":
            ps = 64
            pps = -(-cap // ps)
            bt = rng.permutation(batch * pps).astype(np.int32).reshape(batch, pps)
            kw.update(block_table=bt, page_size=ps, num_pages=batch * pps)
        plan = la.Plan(batch, hkv * g, hkv, 128, lens0, **kw)
        launch = plan.info.grid
        for step in range(3):
            lens = _lens(rng, batch, hi=cap)
            plan.update(lens)
            fresh_kw = dict(kw)
            if schedule != "sequential":
                fresh_kw["grid"] = min(launch, plan.info.total_iters)
            fresh = la.Plan(batch, hkv * g, hkv, 128, lens, **fresh_kw)
            assert np.array_equal(plan.export(), fresh.export()), (trial, step)
            assert plan.info.total_iters == fresh.info.total_iters
            assert plan.info.grid == launch                    # the launch grid never changes
            assert plan.info.updates == step + 1
            # ... and equals the oracle's own walk (stream-K)
            if schedule == "streamk":
                c_n = []
                for (b, _h) in unit_order(batch, hkv, "packed" if layout == "packed" else "bhsd"):
                    c_n += [-(-lens[b] // tile)] * (-(-g // min(8, g)))
                exp = oracle.stream_k_segments(c_n, plan.info.num_vctas)
                assert np.array_equal(plan.export(), np.array([s.row() for s in exp], np.int32).reshape(-1, 7))


def test_launch_grid_from_capacity(la):
    """A plan built for short contexts but an explicit capacity (max_ctx / paged pool) keeps
    one CTA per SM after updating to long contexts (the launch grid is fixed at la_plan)."""
    p = la.Plan(1, 4, 4, 128, [300], host_only=True, max_ctx=1 << 18)
    assert p.info.grid == 148 and p.info.num_vctas == 12          # I = 4 * 3 LeanTiles
    p.update([1 << 18])
    assert p.info.grid == 148 and p.info.num_vctas == 148
    q = la.Plan(1, 4, 4, 128, [300], host_only=True)              # no capacity given: I of the first lens
    assert q.info.grid == 12


def test_update_validation(la):
    p = la.Plan(2, 4, 4, 128, [100, 200], host_only=True, max_ctx=256)
    for lens in ([0, 10], [10, 257], [-1, 5]):
        with pytest.raises(la.LaError) as e:
            p.update(lens)
        assert e.value.status == la.LA_ERR_INVALID
    with pytest.raises(la.LaError) as e:
        p.update([10, 10], block_table=np.zeros((2, 4), np.int32))   # not a paged plan
    assert e.value.status == la.LA_ERR_INVALID
    with pytest.raises(la.LaError) as e:                               # ... nor at la_plan
        la.Plan(2, 4, 4, 128, [100, 200], host_only=True, block_table=np.zeros((2, 4), np.int32), page_size=64,
                num_pages=8)
    assert e.value.status == la.LA_ERR_INVALID
    q = la.Plan(2, 4, 4, 128, [100, 200], host_only=True, q_len=3, causal=True)
    with pytest.raises(la.LaError):
        q.update([2, 100])                                            # n_b < N_b
    before = p.export()
    with pytest.raises(la.LaError):
        p.update([1, 1000])
    assert np.array_equal(p.export(), before) and p.info.updates == 0  # a failed update changes nothing
    pr = synth.Problem(2, 4, 4, 128, [100, 40], layout="paged", page_size=16)
    bt, npages = synth.paged_meta(pr)
    pp = la.Plan(2, 4, 4, 128, pr.ctx_lens, host_only=True, layout="paged", block_table=bt, page_size=16,
                 num_pages=npages)
    bad = bt.copy()
    bad[0, 0] = npages
    with pytest.raises(la.LaError):
        pp.update([100, 40], block_table=bad)
    with pytest.raises(la.LaError):
        pp.update([bt.shape[1] * 16 + 1, 40])                         # beyond the pages of a sequence


def _dynamic_counter_keys(rows, slot_stride, fixed=True):
    """The r01 kernel's fold-tree counter index of every counted segment (groups of 16
    segments from the unit's host; index g0, plus slot_stride for a unit's first group when
    `fixed`).  Returns {index: {(unit, g0), ...}} -- kept to show the shapes where the r01
    indexing collided; r02 folds each unit by its last arriving piece, with ONE
    counter per unit."""
    host = {int(r[1]): int(r[0]) for r in rows if r[4] == 1}
    keys = {}
    for r in rows:
        v, u, h, f = int(r[0]), int(r[1]), int(r[4]), int(r[5])
        if h and f:
            continue                      # one CTA computed the whole unit: nothing is counted
        fhv = host[u]
        g0 = fhv + ((v - fhv) // 16) * 16
        idx = g0 + (slot_stride if (fixed and g0 == fhv) else 0)
        keys.setdefault(idx, set()).add((u, g0))
    return keys


def test_dynamic_pieces_of_a_unit_are_contiguous(la):
    """The kernel's dynamic fold counts a unit's pieces in ONE per-unit counter and expects
    last_cta - host_cta + 1 of them: every virtual CTA from the unit's host to its last CTA
    holds exactly one segment of the unit."""
    rng = np.random.default_rng(5)
    for trial in range(200):
        batch = int(rng.integers(1, 5))
        hkv = int(rng.choice([1, 2, 4, 8]))
        g = int(rng.choice([1, 2, 4, 8]))
        p = la.Plan(batch, hkv * g, hkv, 128, _lens(rng, batch, 1000, 40000), host_only=True, schedule="dynamic",
                    engine="mma", dyn_first_permille=int(rng.integers(500, 1001)))
        rows = p.export()
        for u in np.unique(rows[:, 1]):
            r = rows[rows[:, 1] == u]
            host = int(r[r[:, 4] == 1][0, 0])
            assert sorted(r[:, 0].tolist()) == list(range(host, int(r[0, 6]) + 1))


def test_quantization_efficiency_matches_oracle(la):
    rng = np.random.default_rng(9)
    for trial in range(30):
        batch = int(rng.integers(1, 9))
        heads = int(rng.integers(1, 33))
        lens = _lens(rng, batch, 1, 30000)
        c_n = [-(-lens[b] // 128) for (b, _h) in unit_order(batch, heads, "bhsd")]
        G = int(rng.integers(1, 300))
        p = la.Plan(batch, heads, heads, 128, lens, tile_n=128, host_only=True, grid=G, schedule="streamk")
        exp = oracle.quantization_efficiency(oracle.stream_k_segments(c_n, G), G)
        assert p.info.quantization_efficiency == pytest.approx(exp, rel=1e-12)
        f = la.Plan(batch, heads, heads, 128, lens, tile_n=128, host_only=True, num_sms=148, schedule="fixed_split")
        W = f.info.grid
        exp = oracle.quantization_efficiency(oracle.fixed_split_segments(c_n, W, f.info.split), W)
        assert f.info.quantization_efficiency == pytest.approx(exp, rel=1e-12)
    # c2 on 148 SMs: 65,536 LeanTiles -> 442 / 443 per CTA (Eq. 2): QE = 65536 / (148 * 443)
    c2 = synth.config("c2")
    p = la.Plan(1, 32, 32, 128, c2.ctx_lens, host_only=True)
    assert p.info.quantization_efficiency == pytest.approx(65536 / (148 * 443), rel=1e-12)
