"""C-ABI library (CPU side): it loads, exports every symbol include/la.h declares, and its
host planner reproduces the oracle's stream-K enumeration BIT-EXACTLY (BASELINE.json:
"The planner's tile-to-CTA schedule is integer work and must match a reference
enumeration bit-exactly").  No compute calls -- host-only plans need no GPU."""
import itertools
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
from oracle.lean_attention import unit_order

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def la():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as pkg
    pkg.lib()
    return pkg


def test_exports_every_declared_symbol(la):
    header = open(os.path.join(ROOT, "include", "la.h")).read()
    declared = set(re.findall(r"^\s*(?:la_status|void|int64_t|int|const char\*)\s+(la_\w+)\s*\(", header, re.M))
    assert declared == set(la.EXPORTS)
    nm = subprocess.run(["nm", "-D", "--defined-only", la.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (la_\w+)", nm))
    assert declared <= exported, declared - exported
    L = la.lib()
    assert L.la_version() == 1
    assert L.la_status_string(1) == b"LA_ERR_INVALID"


def test_info_struct_and_trace_fields_match_the_header(la):
    """la_plan_info's ctypes mirror lists the header's fields in order, la_plan_info_get on a
    host-only plan fills the last one (sm_weighted), and the binding reads LA_TRACE_FIELDS
    words per CTA."""
    from paper_2405_10480_b200.leanattn import la_plan_info, Plan
    header = open(os.path.join(ROOT, "include", "la.h")).read()
    body = header[header.index("typedef struct {\n  int batch, heads_q"):header.index("} la_plan_info;")]
    fields = []
    for decl in re.findall(r"^\s*(?:int64_t|int|float|double)\s+([\w, ]+);", body, re.M):
        fields += [f.strip() for f in decl.split(",")]
    assert fields == [f for f, _ in la_plan_info._fields_]
    assert int(re.search(r"#define LA_TRACE_FIELDS (\d+)", header).group(1)) == Plan.TRACE_FIELDS
    p = la.Plan(1, 2, 2, 128, [5000], host_only=True, schedule="streamk")
    assert p.info.sm_weighted == 0
    p.set_weights([3] * p.info.grid)
    assert p.info.sm_weighted == 1


def test_plan_opts_struct_matches_the_header(la):
    """The ctypes mirror of la_plan_opts has the C layout: la_plan_opts_init memsets exactly
    sizeof(la_plan_opts) bytes, so it must touch the whole ctypes struct and nothing past it,
    and its defaults must land in the fields of the same names (engine = LA_ENGINE_AUTO)."""
    import ctypes
    from paper_2405_10480_b200.leanattn import la_plan_opts
    n = ctypes.sizeof(la_plan_opts)
    buf = (ctypes.c_ubyte * (n + 64))(*([0xAB] * (n + 64)))
    assert la.lib().la_plan_opts_init(ctypes.cast(buf, ctypes.POINTER(la_plan_opts))) == 0
    assert all(b == 0xAB for b in bytes(buf)[n:]), "la_plan_opts_init wrote past the ctypes struct"
    o = la_plan_opts.from_buffer(buf)
    assert (o.num_sms, o.ctas_per_sm, o.q_len, o.causal, o.dyn_first_permille, o.engine) == (148, 1, 1, 1, 940, 2)
    header = open(os.path.join(ROOT, "include", "la.h")).read()
    body = header[header.index("typedef struct {\n  float scale;"):header.index("} la_plan_opts;")]
    fields = re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(\w+);", body, re.M)
    assert fields == [f for f, _ in la_plan_opts._fields_]


def _oracle_rows(batch, heads_kv, lens, tile_n, grid, layout):
    units = unit_order(batch, heads_kv, layout)
    c_n = [-(-lens[b] // tile_n) for (b, _h) in units]
    return np.array([s.row() for s in oracle.stream_k_segments(c_n, grid)], dtype=np.int32).reshape(-1, 7)


def test_fig1_golden_through_the_abi(la):
    p = la.Plan(1, 2, 2, 128, [5 * 128], tile_n=128, grid=5, host_only=True, schedule="streamk")
    rows = p.export()
    golden = [tuple(int(x) for x in l.split()) for l in open(os.path.join(ROOT, "tests", "golden", "fig1_schedule.txt"))
              if l.strip() and not l.startswith("#")]
    assert [tuple(r) for r in rows] == golden
    assert p.info.total_iters == 10 and p.info.num_partials == 4 and p.info.grid == 5


def test_exhaustive_small_bit_exact(la):
    n = 0
    for batch, heads, layout in itertools.product([1, 2, 3], [1, 2], ["bhsd", "packed"]):
        for lens in itertools.product([1, 16, 17, 40, 64], repeat=batch):
            I = sum(-(-x // 16) for x in lens) * heads
            for G in sorted({1, 2, 3, I // 2 + 1, I, I + 2}):
                p = la.Plan(batch, heads, heads, 64, list(lens), tile_n=16, grid=G, layout=layout, host_only=True,
                            schedule="streamk")
                got = p.export()
                exp = _oracle_rows(batch, heads, list(lens), 16, G, layout)
                assert np.array_equal(got, exp), (batch, heads, lens, G, layout)
                assert p.info.total_iters == I
                n += 1
    assert n > 500


def test_random_large_and_configs_bit_exact(la):
    rng = np.random.default_rng(0)
    for trial in range(30):
        batch = int(rng.integers(1, 17))
        heads = int(rng.integers(1, 33))
        lens = [int(x) for x in rng.integers(1, 20000, size=batch)]
        tile = int(rng.choice([32, 64, 128, 256]))
        layout = ["bhsd", "packed"][trial % 2]
        I = sum(-(-x // tile) for x in lens) * heads
        G = int(rng.integers(1, min(I, 600) + 1))
        p = la.Plan(batch, heads, heads, 128, lens, tile_n=tile, grid=G, layout=layout, host_only=True,
                    schedule="streamk")
        assert np.array_equal(p.export(), _oracle_rows(batch, heads, lens, tile, G, layout))
    # BASELINE.json configs on a 148-SM B200 (1 CTA / SM)
    import synth
    expect_I = {"c2": 65536, "c3": 32768, "c4": 245056, "c5": 262144}
    for name, I in expect_I.items():
        pr = synth.config(name)
        p = la.Plan(pr.batch, pr.heads_q, pr.heads_kv, pr.head_dim, pr.ctx_lens, tile_n=128, host_only=True,
                    num_sms=148, ctas_per_sm=1, layout=pr.layout, schedule="streamk")
        assert p.info.total_iters == I and p.info.grid == 148 and p.info.tile_n == 128
        rows = p.export()
        assert np.array_equal(rows, _oracle_rows(pr.batch, pr.heads_kv, pr.ctx_lens, 128, 148, pr.layout))
        per = np.bincount(rows[:, 0], weights=rows[:, 3] - rows[:, 2])
        assert per.max() - per.min() <= 1                      # Eq. 2 balance
        # <= 1 partial per CTA (the plan allocates one slot per CTA)
        assert np.bincount(rows[rows[:, 4] == 0][:, 0], minlength=148).max() <= 1
    # c4 packed layout: heads -> total context
    pr = synth.config("c4", layout="packed")
    p = la.Plan(pr.batch, pr.heads_q, pr.heads_kv, pr.head_dim, pr.ctx_lens, tile_n=128, host_only=True,
                layout="packed", schedule="streamk")
    assert np.array_equal(p.export(), _oracle_rows(pr.batch, pr.heads_kv, pr.ctx_lens, 128, 148, "packed"))


def test_auto_tile_and_sequential(la):
    p = la.Plan(1, 32, 32, 128, [262144], host_only=True, schedule="streamk")
    assert p.info.tile_n == 128 and p.info.grid == 148           # P:396 for d=128
    p = la.Plan(1, 8, 8, 64, [1 << 16], host_only=True)
    assert p.info.tile_n == 256                                  # P:396 for d=64
    p = la.Plan(1, 1, 1, 64, [4096], dtype="fp32", host_only=True)
    assert p.info.tile_n == 128 and p.info.grid == 32            # 64 KiB LeanTiles, not split further
    p = la.Plan(2, 3, 3, 128, [300, 1000], tile_n=64, host_only=True, schedule="sequential")
    rows = p.export()
    assert p.info.grid == 6 and len(rows) == 6
    assert all(r[4] == 1 and r[5] == 1 and r[0] == r[1] for r in rows)   # FA2: one full unit per CTA


@pytest.mark.parametrize("args,status", [
    (dict(head_dim=96), 2), (dict(heads_q=3, heads_kv=2), 1), (dict(lens=[0]), 1),
    (dict(tile_n=100), 1), (dict(batch=0, lens=[]), 1),
])
def test_validation(la, args, status):
    kw = dict(batch=1, heads_q=2, heads_kv=2, head_dim=128, lens=[100], tile_n=0)
    kw.update(args)
    with pytest.raises(la.LaError) as e:
        la.Plan(kw["batch"], kw["heads_q"], kw["heads_kv"], kw["head_dim"], kw["lens"], tile_n=kw["tile_n"],
                host_only=True)
    assert e.value.status == status


def test_dynamic_schedule_bit_exact(la):
    """LA_SCHED_DYNAMIC: Alg. 2's walk over the balanced virtual-CTA ranges (heads + tail
    chunks), bit-exact against the oracle's layout, incl. the claim order (la_plan_export's
    rows are per virtual CTA; the claim order is checked through la_plan_info + the oracle)."""
    rng = np.random.default_rng(1)
    import synth
    cases = [(synth.config(c), 148, 940, 2) for c in ("c2", "c3", "c4", "c5")]
    for trial in range(25):
        batch = int(rng.integers(1, 9))
        heads = int(rng.integers(1, 17))
        lens = [int(x) for x in rng.integers(1, 30000, size=batch)]
        cases.append((synth.Problem(batch, heads, heads, 128, lens, layout=["bhsd", "packed"][trial % 2]),
                      int(rng.integers(1, 200)), int(rng.integers(500, 1001)), int(rng.integers(1, 6))))
    for pr, sms, hp, mc in cases:
        p = la.Plan(pr.batch, pr.heads_q, pr.heads_kv, pr.head_dim, pr.ctx_lens, tile_n=128, host_only=True,
                    num_sms=sms, layout=pr.layout, schedule="dynamic", dyn_first_permille=hp, dyn_min_chunk=mc)
        units = unit_order(pr.batch, pr.heads_kv, pr.layout)
        c_n = [-(-pr.ctx_lens[b] // 128) for (b, _h) in units]
        I = sum(c_n)
        G = min(sms, I)
        begins, claim = oracle.balanced_ranges(I, G, hp, mc)
        exp = np.array([s.row() for s in oracle.segments_from_ranges(c_n, begins)], dtype=np.int32).reshape(-1, 7)
        assert np.array_equal(p.export(), exp)
        assert p.info.num_vctas == len(begins) - 1 and p.info.grid == G
        assert p.info.num_vctas <= p.info.slot_capacity
        assert p.claims().tolist() == claim
        # partial slots: <= 1 non-host and <= 1 non-finishing-host segment per virtual CTA
        rows = p.export()
        assert np.bincount(rows[rows[:, 4] == 0][:, 0], minlength=p.info.num_vctas).max() <= 1
        wait_hosts = rows[(rows[:, 4] == 1) & (rows[:, 5] == 0)]
        assert np.bincount(wait_hosts[:, 0], minlength=p.info.num_vctas).max() <= 1


def test_weighted_streamk_bit_exact(la):
    """la_plan_set_weights: the SM-rate-weighted stream-K ranges and Alg. 2's walk over them,
    bit-exact against oracle.weighted_ranges + oracle.segments_from_ranges; the weights
    persist across la_plan_update; NULL restores Eq. 2."""
    rng = np.random.default_rng(3)
    import synth
    cases = [synth.config(c) for c in ("c2", "c3", "c4")]
    for trial in range(20):
        batch = int(rng.integers(1, 9))
        hkv = int(rng.integers(1, 9))
        lens = [int(x) for x in rng.integers(1, 30000, size=batch)]
        cases.append(synth.Problem(batch, hkv * int(rng.integers(1, 3)), hkv, 128, lens,
                                   layout=["bhsd", "packed"][trial % 2]))
    for i, pr in enumerate(cases):
        sms = [148, 37, 200, 5][i % 4]
        p = la.Plan(pr.batch, pr.heads_q, pr.heads_kv, pr.head_dim, pr.ctx_lens, tile_n=128, host_only=True,
                    num_sms=sms, layout=pr.layout, schedule="streamk")
        G = p.info.grid
        w = [int(x) for x in rng.integers(1, 1 << 20, size=G)] if i % 2 else \
            [int(x) for x in rng.integers(60000, 70000, size=G)]
        p.set_weights(w)
        assert p.info.sm_weighted == 1
        units = unit_order(pr.batch, pr.heads_kv, pr.layout)
        c_n = [-(-pr.ctx_lens[b] // 128) for (b, _h) in units for _ in range(-(-pr.group // 8))]
        begins = oracle.weighted_ranges(sum(c_n), w)
        exp = np.array([s.row() for s in oracle.segments_from_ranges(c_n, begins)], dtype=np.int32).reshape(-1, 7)
        assert np.array_equal(p.export(), exp)
        rows = p.export()   # <= 1 non-host and <= 1 waiting-host segment per CTA (any contiguous ranges)
        assert np.bincount(rows[rows[:, 4] == 0][:, 0], minlength=G).max(initial=0) <= 1
        wait_hosts = rows[(rows[:, 4] == 1) & (rows[:, 5] == 0)]
        assert np.bincount(wait_hosts[:, 0], minlength=G).max(initial=0) <= 1
        # the weights stay with the plan across an update (per CTA, independent of ctx_lens)
        lens2 = [max(1, n // 2 + 7) for n in pr.ctx_lens]
        p.update(lens2)
        c_n2 = [-(-n // 128) for (b, _h) in units for n in [lens2[b]] for _ in range(-(-pr.group // 8))]
        begins2 = oracle.weighted_ranges(sum(c_n2), w[:min(G, sum(c_n2))])
        exp2 = np.array([s.row() for s in oracle.segments_from_ranges(c_n2, begins2)], dtype=np.int32).reshape(-1, 7)
        assert np.array_equal(p.export(), exp2)
        p.set_weights(None)
        assert p.info.sm_weighted == 0
        exp3 = np.array([s.row() for s in oracle.stream_k_segments(c_n2, min(G, sum(c_n2)))],
                        dtype=np.int32).reshape(-1, 7)
        assert np.array_equal(p.export(), exp3)
    # validation: wrong count, out-of-range weight, non-stream-K plan
    p = la.Plan(1, 2, 2, 128, [5000], host_only=True, schedule="streamk")
    for bad in ([1] * (p.info.grid + 1), [0] * p.info.grid, [(1 << 20) + 1] * p.info.grid):
        with pytest.raises(la.LaError) as e:
            p.set_weights(bad)
        assert e.value.status == la.LA_ERR_INVALID
    pd = la.Plan(1, 2, 2, 128, [5000], host_only=True, schedule="dynamic")
    with pytest.raises(la.LaError) as e:
        pd.set_weights([1] * pd.info.grid)
    assert e.value.status == la.LA_ERR_STATE


def test_fixed_split_schedule_bit_exact(la):
    """LA_SCHED_FIXED_SPLIT (NEXT-1, FlashDecoding's decomposition): chunk ranges and the
    FA2 split heuristic, bit-exact against the oracle."""
    import synth
    rng = np.random.default_rng(2)
    cases = [(synth.Problem(1, 56, 56, 64, [262144]), 0), (synth.Problem(4, 32, 32, 128, [262144] * 4), 0),
             (synth.config("c2"), 0), (synth.config("c4"), 3)]
    for trial in range(20):
        batch = int(rng.integers(1, 9))
        heads = int(rng.integers(1, 17))
        lens = [int(x) for x in rng.integers(1, 30000, size=batch)]
        cases.append((synth.Problem(batch, heads, heads, 128, lens), int(rng.integers(0, 9))))
    for pr, split in cases:
        p = la.Plan(pr.batch, pr.heads_q, pr.heads_kv, pr.head_dim, pr.ctx_lens, tile_n=128, host_only=True,
                    num_sms=148, layout=pr.layout, schedule="fixed_split", split=split)
        units = unit_order(pr.batch, pr.heads_kv, pr.layout)
        c_n = [-(-pr.ctx_lens[b] // 128) for (b, _h) in units]
        s = split or oracle.fa2_num_splits(len(c_n), max(c_n), 148)
        assert p.info.split == s
        begins = oracle.fixed_split_ranges(c_n, s)
        exp = np.array([x.row() for x in oracle.segments_from_ranges(c_n, begins)], dtype=np.int32).reshape(-1, 7)
        assert np.array_equal(p.export(), exp)
    # the paper's motivating shapes: 56 heads x batch 1 -> FD splits; batch 4 x
    # 32 heads fills 80% of 148 SMs -> no split at all (one partial wave)
    assert oracle.fa2_num_splits(56, 2048, 148) > 1 and oracle.fa2_num_splits(128, 2048, 148) == 1


def test_paged_plan_validation_and_schedule(la):
    import synth
    p = synth.Problem(3, 4, 4, 128, [100, 17, 640], layout="paged", page_size=16)
    bt, npages = synth.paged_meta(p)
    plan = la.Plan(3, 4, 4, 128, p.ctx_lens, tile_n=64, host_only=True, layout="paged", block_table=bt,
                   page_size=16, num_pages=npages, schedule="streamk", grid=7)
    ref = la.Plan(3, 4, 4, 128, p.ctx_lens, tile_n=64, host_only=True, schedule="streamk", grid=7)
    assert np.array_equal(plan.export(), ref.export())      # units batch -> heads, like BHSD
    for bad in (dict(page_size=24), dict(num_pages=3), dict(page_size=16, block_table=bt[:, :2])):
        kw = dict(block_table=bt, page_size=16, num_pages=npages)
        kw.update(bad)
        with pytest.raises(la.LaError):
            la.Plan(3, 4, 4, 128, p.ctx_lens, host_only=True, layout="paged", **kw)


def test_xchg_validation(la):
    """NEXT-2 exchange options are validated at la_plan (host-only plans: no buffer)."""
    for kw, status in [(dict(xchg_world=9), la.LA_ERR_INVALID), (dict(xchg_world=2, xchg_rank=2), la.LA_ERR_INVALID),
                       (dict(xchg_world=2, xchg_rank=-1), la.LA_ERR_INVALID),
                       (dict(xchg_world=2, q_len=2), la.LA_ERR_UNSUPPORTED)]:
        with pytest.raises(la.LaError) as e:
            la.Plan(1, 2, 2, 128, [100], host_only=True, **kw)
        assert e.value.status == status, kw
    p = la.Plan(1, 2, 2, 128, [100], host_only=True, xchg_world=4, xchg_rank=3)
    with pytest.raises(la.LaError) as e:
        p.xchg_handle()
    assert e.value.status == la.LA_ERR_STATE
    la.Plan(1, 2, 2, 128, [100], host_only=True, xchg_world=2, q_len=2, causal=False)  # full mask: shard-local


def test_query_tiles_and_heterogeneous_batches_bit_exact(la):
    """NEXT-3: the g * N_b rows of (b, h_kv) are cut into C_m = ceil(g N_b / T_m) query
    tiles (Alg2§4), T_m = min(8, max_b g N_b); each tile is a unit streaming the whole KV of
    (b, h_kv), tiles innermost in the memory-order linearisation (C14).  The planner's
    segments must equal the oracle's stream-K walk over that unit list, bit for bit."""
    rng = np.random.default_rng(5)
    for trial in range(40):
        batch = int(rng.integers(1, 6))
        hkv = int(rng.integers(1, 4))
        g = int(rng.choice([1, 2, 3, 4, 8, 16]))
        lens = [int(x) for x in rng.integers(16, 3000, size=batch)]
        qls = [int(x) for x in rng.integers(1, 6, size=batch)]
        layout = ["bhsd", "packed"][trial % 2]
        tile = int(rng.choice([32, 64, 128]))
        engine = ["mma", "tcgen05", "auto"][(trial // 2) % 3]
        p = la.Plan(batch, hkv * g, hkv, 128, lens, tile_n=tile, grid=int(rng.integers(1, 300)), layout=layout,
                    host_only=True, schedule="streamk", q_lens=qls, engine=engine)
        tm = min(8 if engine == "mma" else 32, max(g * n for n in qls))
        c_n = []
        for (b, _h) in unit_order(batch, hkv, layout):
            c_n += [-(-lens[b] // tile)] * (-(-(g * qls[b]) // tm))
        exp = np.array([s.row() for s in oracle.stream_k_segments(c_n, p.info.grid)], dtype=np.int32).reshape(-1, 7)
        assert np.array_equal(p.export(), exp), trial
        assert p.info.tile_rows == tm and p.info.num_units == len(c_n)
        assert p.info.q_rows == sum(hkv * g * n for n in qls)
        assert p.info.q_len == (qls[0] if len(set(qls)) == 1 else 0)


def test_heterogeneous_validation(la):
    for qls, status in [([1, 0], la.LA_ERR_INVALID), ([1, 101], la.LA_ERR_INVALID)]:
        with pytest.raises(la.LaError) as e:
            la.Plan(2, 2, 2, 128, [100, 100], host_only=True, q_lens=qls)
        assert e.value.status == status
    with pytest.raises(la.LaError) as e:   # causal multi-token blocks are not shard-local
        la.Plan(2, 2, 2, 128, [100, 100], host_only=True, q_lens=[1, 2], xchg_world=2)
    assert e.value.status == la.LA_ERR_UNSUPPORTED
    p = la.Plan(1, 32, 2, 128, [1000], host_only=True, engine="mma")  # MQA-like g = 16: two 8-row tiles
    assert p.info.tile_rows == 8 and p.info.num_units == 4
    p = la.Plan(1, 32, 2, 128, [1000], host_only=True)  # auto: tcgen05's 16-row tiles, one per KV head
    assert p.info.tile_rows == 16 and p.info.num_units == 2
    p = la.Plan(1, 32, 2, 128, [1000], host_only=True, schedule="dynamic")  # auto, dynamic: mma.sync tiles
    assert p.info.tile_rows == 8 and p.info.num_units == 4
    p = la.Plan(1, 16, 2, 128, [1000], host_only=True)  # auto, g = 8: mma.sync
    assert p.info.tile_rows == 8 and p.info.num_units == 2


def test_fp8_plan(la):
    # FP8 KV (NEXT-4): 64 KiB LeanTiles are 256 tokens at d = 128; d = 64 is not built
    p = la.Plan(1, 32, 32, 128, [262144], dtype="fp8", host_only=True)
    assert p.info.tile_n == 256 and p.info.grid == 148 and p.info.kv_bytes == 2 * 32 * 262144 * 128
    with pytest.raises(la.LaError) as e:
        la.Plan(1, 2, 2, 64, [100], dtype="fp8", host_only=True)
    assert e.value.status == 2
    with pytest.raises(la.LaError) as e:
        la.Plan(1, 2, 2, 128, [100], dtype="fp8", host_only=True, k_scale=-1.0)
    assert e.value.status == 1
