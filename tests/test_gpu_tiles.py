"""NEXT-3 completed: query tiles (C_m > 1: any group size, g * N_q > 8, e.g. MQA) and
heterogeneous batches (per-request N_b: decode mixed with speculative / chunked-prefill
blocks), through the C-ABI, against the fp64 oracle on the same seeded inputs."""
import numpy as np
import pytest
import torch

import oracle
import synth
from _helpers import gate

pytestmark = pytest.mark.gpu


def _oracle(p, causal=True):
    q = synth.to_f64(synth.gen_q(p)).reshape(-1, p.head_dim)
    k = synth.to_f64(synth.fill_kv_cache(p, "k"))
    v = synth.to_f64(synth.fill_kv_cache(p, "v"))
    qls = list(p.q_lens) if p.q_lens is not None else [p.q_len] * p.batch
    bt = synth.paged_meta(p)[0] if p.layout == "paged" else None
    return oracle.decode_attention_varq(q, k, v, p.ctx_lens, qls, p.scale, causal, p.layout, block_table=bt,
                                        page_size=p.page_size)


def _cuda(p, causal=True, **kw):
    import paper_2405_10480_b200 as la
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    extra = {}
    if p.layout == "paged":
        bt, num_pages = synth.paged_meta(p)
        extra = dict(block_table=bt, page_size=p.page_size, num_pages=num_pages)
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, layout=p.layout,
                   q_len=p.q_len, q_lens=p.q_lens, causal=causal, **extra, **kw)
    out, lse = plan.decode(q, k, v)
    torch.cuda.synchronize()
    return out.reshape(-1, p.head_dim).cpu().numpy(), lse.reshape(-1).cpu().numpy(), plan


@pytest.mark.parametrize("engine", ["mma", "auto"])
@pytest.mark.parametrize("hq,hkv,d", [(32, 2, 128), (16, 1, 64), (24, 2, 128)])
def test_large_groups_mqa(hq, hkv, d, engine):
    """g = 16, 16, 12 with N_q = 1: C_m = 2 query tiles of 8 rows per KV head on mma.sync
    (g > 8 was unsupported); "auto" takes the tcgen05 engine's 16-row tiles (C_m = 1) at d = 128."""
    p = synth.Problem(2, hq, hkv, d, [1500, 2777], dtype="bf16", dist="D2", seed=81)
    O, L, plan = _cuda(p, engine=engine)
    tm = 32 if engine == "auto" and d == 128 else 8
    g = hq // hkv
    assert plan.info.tile_rows == min(tm, g) and plan.info.num_units == 2 * hkv * -(-g // tm)
    assert plan.info.engine == (1 if tm == 32 else 0)
    gate(O, L, *_oracle(p), what=f"g={g} {engine}")


@pytest.mark.parametrize("engine", ["mma", "auto"])
@pytest.mark.parametrize("causal", [True, False])
def test_query_tiles_multi_token(causal, engine):
    """g = 8 x N_q = 3 = 24 rows -> 3 tiles of 8 (mma.sync) or one of 24 (tcgen05 via "auto");
    the causal limit follows the row's query index."""
    p = synth.Problem(2, 16, 2, 128, [900, 2000], dtype="bf16", dist="D1", seed=82, q_len=3)
    O, L, plan = _cuda(p, causal=causal, engine=engine)
    assert plan.info.num_units == 2 * 2 * (3 if engine == "mma" else 1)
    gate(O, L, *_oracle(p, causal), what=f"tiles causal={causal} {engine}")


@pytest.mark.parametrize("dtype,d", [("bf16", 128), ("fp16", 64)])
@pytest.mark.parametrize("causal", [True, False])
def test_heterogeneous_batch(dtype, d, causal):
    """Per-request N_b (decode rows next to 5- and 8-token blocks), g = 2."""
    p = synth.Problem(4, 8, 4, d, [700, 3000, 1234, 64], dtype=dtype, dist="D2", seed=83, q_lens=[1, 5, 2, 8])
    O, L, plan = _cuda(p, causal=causal)
    assert plan.info.q_len == 0 and plan.info.q_rows == 8 * 16
    gate(O, L, *_oracle(p, causal), what=f"hetero {dtype} causal={causal}")


def test_heterogeneous_mha_rows_and_packed():
    """g = 1 with N_b in {1, 3}: rows > 1 somewhere -> tensor-core engine for all; packed KV."""
    p = synth.Problem(3, 4, 4, 128, [333, 4096, 1000], dtype="bf16", dist="D1", seed=84, q_lens=[1, 3, 1],
                      layout="packed")
    O, L, _ = _cuda(p)
    gate(O, L, *_oracle(p), what="hetero g=1 packed")


def test_heterogeneous_paged():
    p = synth.Problem(2, 16, 2, 128, [1000, 2500], dtype="bf16", dist="D1", seed=85, q_lens=[2, 1],
                      layout="paged", page_size=32)
    O, L, _ = _cuda(p)
    gate(O, L, *_oracle(p), what="hetero paged")


@pytest.mark.parametrize("schedule", ["streamk", "dynamic", "fixed_split", "sequential"])
def test_tiles_every_schedule_deterministic(schedule):
    p = synth.Problem(2, 32, 2, 128, [5000, 3001], dtype="bf16", dist="D1", seed=86, q_lens=[1, 2])
    ref = _oracle(p)
    O0, L0, _ = _cuda(p, schedule=schedule, grid=37)
    gate(O0, L0, *ref, what=f"tiles {schedule}")
    for _ in range(3):
        O, L, _ = _cuda(p, schedule=schedule, grid=37)
        assert np.array_equal(O, O0) and np.array_equal(L, L0)
