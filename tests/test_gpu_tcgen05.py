"""GPU parity of the tcgen05 engine (LA_ENGINE_TCGEN05: 5th-gen tensor cores, S^T and the
per-stage O^T in TMEM) against the fp64 oracle -- the same gates and cases as the mma.sync
GQA engine: groups 2..8, N_q > 1 (causal or full), ragged tails, tile sizes below, at and
above one 128-token stage, every schedule, packed layout, determinism, c3 at full size."""
import numpy as np
import pytest
import torch

import synth
from _helpers import census_expect, cuda_inputs, gate, oracle_unit, run_cuda, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as la
    la.lib()


TC5 = dict(engine="tcgen05")


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("group", [2, 4, 8])
def test_tcgen05_small_multi_tile_ragged(dtype, group):
    p = synth.Problem(2, 2 * group, 2, 128, [1000, 777], dtype=dtype, dist="D2", seed=31, max_ctx=1024)
    O_ref, L_ref = run_oracle(p)
    inputs = cuda_inputs(p)
    for schedule in ("streamk", "dynamic", "fixed_split", "sequential"):
        for tile_n in (64, 128, 256):
            for grid in (1, 3, 0):
                O, L, _ = run_cuda(p, inputs=inputs, tile_n=tile_n, grid=grid, schedule=schedule, **TC5)
                gate(O, L, O_ref, L_ref, what=f"tc5 g{group}/{dtype}/T{tile_n}/G{grid}/{schedule}")


@pytest.mark.parametrize("dist", ["D0", "D1", "D3", "D4"])
def test_tcgen05_distributions_packed(dist):
    p = synth.Problem(3, 16, 2, 128, [700, 1500, 64], dtype="bf16", dist=dist, seed=32, layout="packed")
    O_ref, L_ref = run_oracle(p)
    O, L, _ = run_cuda(p, tile_n=128, grid=0, **TC5)
    gate(O, L, O_ref, L_ref, what=f"tc5 packed {dist}")


@pytest.mark.parametrize("group,q_len", [(1, 2), (1, 8), (2, 4), (4, 2)])
@pytest.mark.parametrize("causal", [True, False])
def test_tcgen05_multi_token(group, q_len, causal):
    p = synth.Problem(2, 2 * group, 2, 128, [900, 333], dtype="bf16", dist="D2", seed=61, q_len=q_len)
    O_ref, L_ref = run_oracle(p, causal=causal)
    inputs = cuda_inputs(p)
    for schedule in ("streamk", "dynamic"):
        for tile_n, grid in ((128, 7), (128, 0)):
            O, L, _ = run_cuda(p, inputs=inputs, tile_n=tile_n, grid=grid, schedule=schedule, causal=causal, **TC5)
            gate(O, L, O_ref, L_ref, what=f"tc5 Nq{q_len} g{group} causal={causal} G{grid} {schedule}")


def test_tcgen05_determinism_and_equivalence():
    import paper_2405_10480_b200 as la
    p = synth.Problem(1, 8, 1, 128, [5000], dtype="bf16", dist="D2", seed=33)
    q, k, v = cuda_inputs(p)
    for schedule in ("streamk", "dynamic"):
        plan = la.Plan(1, 8, 1, 128, [5000], grid=11, tile_n=128, schedule=schedule, engine="tcgen05")
        ref = plan.decode(q, k, v)[0].clone()
        for _ in range(5):
            assert torch.equal(plan.decode(q, k, v)[0], ref)
        mma = la.Plan(1, 8, 1, 128, [5000], grid=11, tile_n=128, schedule=schedule, engine="mma").decode(q, k, v)[0]
        assert (ref - mma).abs().max().item() <= 2e-5  # both engines: P = P_hi + P_lo, fp32 sums


def test_tcgen05_plan_errors():
    import paper_2405_10480_b200 as la
    with pytest.raises(la.LaError):  # FP8 caches stay on their f16 mma.sync engine
        la.Plan(1, 8, 1, 128, [1000], engine="tcgen05", dtype="fp8", k_scale=1.0, v_scale=1.0)
    plan = la.Plan(1, 4, 4, 128, [1000], engine="tcgen05")  # MHA (T_m = 1): CUDA cores, engine ignored
    assert plan.info.group == 1


def test_tcgen05_c3_full_size_sampled():
    """BASELINE.json config 3 on the tcgen05 engine, sampled units + census closed form."""
    p = synth.config("c3")
    inputs = cuda_inputs(p)
    refs = {(b, h): oracle_unit(p, b, h) for b, h in ((0, 0), (3, 5), (7, 7))}
    for schedule in ("streamk", "dynamic"):
        O, L, plan = run_cuda(p, inputs=inputs, schedule=schedule, **TC5)
        assert plan.info.total_iters == 32768 and plan.info.group == 8
        for (b, h), (O_ref, L_ref) in refs.items():
            gate(O[b, 8 * h:8 * h + 8], L[b, 8 * h:8 * h + 8], O_ref, L_ref, what=f"tc5 c3 b{b} h{h} {schedule}")
    del inputs
    torch.cuda.empty_cache()
    p3 = synth.config("c3", dist="D3")
    O3, L3, _ = run_cuda(p3, **TC5)
    o_exp, l_exp = census_expect(p3, 0)
    assert np.max(np.abs(O3 - o_exp[None, None, :])) <= 1e-5
    assert np.max(np.abs(L3 - l_exp)) <= 1e-5


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("heads_q,heads_kv,q_len,causal", [(32, 2, 1, True), (16, 1, 1, True), (24, 2, 1, True),
                                                           (16, 2, 2, True), (16, 2, 2, False), (8, 1, 3, True),
                                                           (32, 1, 1, True), (16, 2, 4, True), (24, 1, 2, True),
                                                           (40, 2, 1, True), (16, 2, 4, False)])
def test_tcgen05_wide_tiles(dtype, heads_q, heads_kv, q_len, causal):
    """16- and 32-row query tiles (the tcgen05 engine's N = 16 / 32): g * N_q rows of a KV head
    in ONE pass where mma.sync tiles take two to four (g = 16, MQA 16 / 32, g = 12, g = 20,
    g = 8 x N_q 2 / 3 / 4, g = 24 x N_q 2 -> 32 + 16 rows)."""
    p = synth.Problem(2, heads_q, heads_kv, 128, [1000, 333], dtype=dtype, dist="D2", seed=71, q_len=q_len)
    O_ref, L_ref = run_oracle(p, causal=causal)
    inputs = cuda_inputs(p)
    for schedule in ("streamk", "sequential"):
        for tile_n, grid in ((128, 5), (256, 0)):
            O, L, plan = run_cuda(p, inputs=inputs, tile_n=tile_n, grid=grid, schedule=schedule, causal=causal, **TC5)
            assert plan.info.tile_rows == min(32, p.group * q_len)
            gate(O, L, O_ref, L_ref, what=f"tc5 wide H{heads_q}/{heads_kv} Nq{q_len} {dtype} {schedule} G{grid}")


def test_tcgen05_wide_tiles_one_kv_pass_and_rejects_dynamic():
    import paper_2405_10480_b200 as la
    wide = la.Plan(2, 32, 2, 128, [4096, 4096], engine="tcgen05", host_only=True)
    narrow = la.Plan(2, 32, 2, 128, [4096, 4096], host_only=True, engine="mma")
    assert wide.info.num_units == 4 and narrow.info.num_units == 8  # C_m = 1 vs 2 query tiles per KV head
    with pytest.raises(la.LaError):
        la.Plan(2, 32, 2, 128, [4096, 4096], engine="tcgen05", schedule="dynamic")


def test_tcgen05_wide_c3_speculative_full_size():
    """c3 with N_q = 2 (speculative decode: 16 rows per KV head, ONE pass over the cache) vs the
    oracle-pinned mma.sync engine (two 8-row passes) at full size, and the census closed form."""
    p = synth.config("c3", q_len=2)
    inputs = cuda_inputs(p)
    O, L, plan = run_cuda(p, inputs=inputs, **TC5)
    assert plan.info.tile_rows == 16 and plan.info.num_units == 64
    import oracle
    q64 = synth.to_f64(synth.gen_q(p))
    for b, h in ((0, 0), (5, 3)):  # sampled units: 8 heads x 2 queries against the oracle
        k = synth.to_f64(synth.gen_kv_unit(p, b, h, "k"))[None, None]
        v = synth.to_f64(synth.gen_kv_unit(p, b, h, "v"))[None, None]
        O_ref, L_ref = oracle.decode_attention_multi(q64[b:b + 1, 8 * h:8 * h + 8], k, v, [p.ctx_lens[b]], p.scale)
        gate(O[b:b + 1, 8 * h:8 * h + 8], L[b:b + 1, 8 * h:8 * h + 8], O_ref, L_ref, what=f"tc5 c3 Nq2 b{b} h{h}")
    O2, L2, plan2 = run_cuda(p, inputs=inputs, engine="mma")
    assert plan2.info.num_units == 128
    assert np.abs(O - O2).max() <= 1e-4 and np.abs(L - L2).max() <= 2e-6  # fp32 sums over 64k keys
    del inputs
    torch.cuda.empty_cache()
    p3 = synth.config("c3", q_len=2, dist="D3")
    O3, L3, _ = run_cuda(p3, causal=False, **TC5)
    o_exp, l_exp = census_expect(p3, 0)
    assert np.max(np.abs(O3 - o_exp)) <= 1e-5
    assert np.max(np.abs(L3 - l_exp)) <= 1e-5
    torch.cuda.empty_cache()


def test_tcgen05_wide_c3_q4_full_size():
    """c3 with N_q = 4 -- the `bench.py --config c3 --q-len 4` launch: 32 rows per KV head in
    ONE pass on the 2-warpgroup / 3-slot engine (stage j -> warpgroup j mod 2, slot j mod 3),
    segments of ~220 stages, vs the oracle on sampled units (causal: query i sees n - 4 + i + 1
    keys) and vs the mma.sync engine (four 8-row passes), plus the census closed form."""
    p = synth.config("c3", q_len=4)
    inputs = cuda_inputs(p)
    O, L, plan = run_cuda(p, inputs=inputs, causal=True, **TC5)
    assert plan.info.tile_rows == 32 and plan.info.num_units == 64
    import oracle
    q64 = synth.to_f64(synth.gen_q(p))
    for b, h in ((0, 0), (7, 5)):  # sampled units: 8 heads x 4 queries against the oracle
        k = synth.to_f64(synth.gen_kv_unit(p, b, h, "k"))[None, None]
        v = synth.to_f64(synth.gen_kv_unit(p, b, h, "v"))[None, None]
        O_ref, L_ref = oracle.decode_attention_multi(q64[b:b + 1, 8 * h:8 * h + 8], k, v, [p.ctx_lens[b]], p.scale,
                                                     causal=True)
        gate(O[b:b + 1, 8 * h:8 * h + 8], L[b:b + 1, 8 * h:8 * h + 8], O_ref, L_ref, what=f"tc5 c3 Nq4 b{b} h{h}")
    O2, L2, plan2 = run_cuda(p, inputs=inputs, causal=True, engine="mma")
    assert plan2.info.num_units == 256
    assert np.abs(O - O2).max() <= 1e-4 and np.abs(L - L2).max() <= 2e-6  # fp32 sums over 64k keys
    del inputs
    torch.cuda.empty_cache()
    p3 = synth.config("c3", q_len=4, dist="D3")
    O3, L3, _ = run_cuda(p3, causal=False, **TC5)
    o_exp, l_exp = census_expect(p3, 0)
    assert np.max(np.abs(O3 - o_exp)) <= 1e-5
    assert np.max(np.abs(L3 - l_exp)) <= 1e-5
    torch.cuda.empty_cache()


@pytest.mark.parametrize("rows", [8, 16, 32])
@pytest.mark.parametrize("page_size", [16, 32, 64, 128, 256])
def test_tcgen05_paged(rows, page_size):
    """Paged pools on the tcgen05 engine: per-half TMA boxes of min(128, page) rows inside one
    page keep the stage's operand layout; 8-row (g = 8) and 16-row (g = 16) tiles."""
    p = synth.Problem(3, 2 * rows, 2, 128, [1000, 77, 2500], dtype="bf16", dist="D2", seed=51,
                      layout="paged", page_size=page_size)
    O_ref, L_ref = run_oracle(p)
    inputs = cuda_inputs(p)
    for schedule in (("streamk", "dynamic") if rows == 8 else ("streamk", "sequential")):
        for tile_n, grid in ((128, 5), (256, 0)):
            O, L, plan = run_cuda(p, inputs=inputs, tile_n=tile_n, grid=grid, schedule=schedule, **TC5)
            assert plan.info.engine == 1 and plan.info.tile_rows == rows
            gate(O, L, O_ref, L_ref, what=f"tc5 paged rows{rows} ps{page_size} T{tile_n} G{grid} {schedule}")


@pytest.mark.parametrize("rows_per_head", [8, 16, 32])
def test_tcgen05_tiny_contexts(rows_per_head):
    """Contexts of 1..129 tokens (one short stage, a stage plus one token) and N_q = 2 blocks
    whose causal limits cut inside the only stage."""
    g = rows_per_head
    p = synth.Problem(4, 2 * g, 2, 128, [1, 3, 128, 129], dtype="bf16", dist="D2", seed=91)
    O_ref, L_ref = run_oracle(p)
    for grid in (1, 0):
        O, L, _ = run_cuda(p, grid=grid, **TC5)
        gate(O, L, O_ref, L_ref, what=f"tc5 tiny g{g} G{grid}")
    p2 = synth.Problem(3, g, 2, 128, [2, 9, 200], dtype="bf16", dist="D2", seed=92, q_len=2)
    O_ref, L_ref = run_oracle(p2, causal=True)
    O, L, plan = run_cuda(p2, causal=True, **TC5)
    assert plan.info.tile_rows == g
    gate(O, L, O_ref, L_ref, what=f"tc5 tiny Nq2 g{g // 2}")


@pytest.mark.parametrize("q_len,n,grid,tile_n", [(4, 40000, 0, 128), (4, 40000, 37, 128), (2, 9000, 0, 32),
                                                 (4, 2000, 148, 16)])
def test_tcgen05_wide_tiles_many_peers(q_len, n, grid, tile_n):
    """One 16 / 32-row unit spread over up to 148 CTAs: the host's peer partials exceed the idle
    ring (147 peers x 32 rows), so its epilogue warps read the peers' rows from L2, while units
    spread over few CTAs stage every peer at once -- both against the oracle."""
    p = synth.Problem(1, 8, 1, 128, [n], dtype="bf16", dist="D2", seed=75, q_len=q_len)
    O_ref, L_ref = run_oracle(p)
    O, L, plan = run_cuda(p, tile_n=tile_n, grid=grid, **TC5)
    assert plan.info.tile_rows == 8 * q_len and plan.info.num_units == 1
    gate(O, L, O_ref, L_ref, what=f"tc5 wide many peers Nq{q_len} n{n} G{plan.info.grid} T{tile_n}")
