"""NEXT-2 fused cross-GPU fixup, exercised on ONE GPU: P "ranks" are P plans in this
process, each decoding its sequence shard on its own stream (grids sized so all P kernels
are co-resident), their exchange buffers attached to each other (la_plan_xchg_attach) --
the same kernel protocol as P GPUs over NVLink (stores into the peers' buffers, release /
acquire flags at system scope), only the buffer addresses differ.  Every rank must return
the FULL attention result, bitwise identical across ranks, within the parity gate of the
oracle on the unsharded problem, over several launches (double-buffer parity)."""
import numpy as np
import pytest
import torch

import synth
from _helpers import gate, run_oracle

pytestmark = pytest.mark.gpu


def _shards(p, world):
    return [synth.shard_bounds(p, r, world) for r in range(world)]


def _run_fused(p, world, schedule="streamk", launches=3, causal=True):
    import paper_2405_10480_b200 as la
    dev = torch.device("cuda")
    q = synth.gen_q(p, dev)
    grid = max(1, 140 // world)
    plans, kv = [], []
    for r, bounds in enumerate(_shards(p, world)):
        lens = [b - a for a, b in bounds]
        kv.append((synth.fill_kv_cache(p, "k", dev, token_range=bounds),
                   synth.fill_kv_cache(p, "v", dev, token_range=bounds)))
        fp8 = dict(k_scale=p.k_scale, v_scale=p.v_scale) if p.dtype == "fp8" else {}
        plans.append(la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, lens, dtype=p.dtype, grid=grid,
                             schedule=schedule, xchg_world=world, xchg_rank=r, q_len=p.q_len, causal=causal,
                             **fp8))
    for r in range(world):
        for s in range(world):
            if s != r:
                plans[r].xchg_attach(s, plans[s])
    streams = [torch.cuda.Stream() for _ in range(world)]
    outs = []
    for it in range(launches):
        torch.cuda.synchronize()
        res = []
        for r in range(world):
            with torch.cuda.stream(streams[r]):
                res.append(plans[r].decode(q, kv[r][0], kv[r][1], stream=streams[r]))
        torch.cuda.synchronize()
        for r in range(world):
            plans[r].xchg_status()
        outs.append([(o.cpu().numpy(), l.cpu().numpy()) for o, l in res])
    return outs


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("schedule", ["streamk", "sequential", "dynamic"])
def test_fused_exchange_mha(world, schedule):
    p = synth.Problem(2, 4, 4, 128, [3000, 5333], dtype="bf16", dist="D2", seed=71)
    O_ref, L_ref = run_oracle(p)
    outs = _run_fused(p, world, schedule)
    for it, per_rank in enumerate(outs):
        O0, L0 = per_rank[0]
        for r, (O, L) in enumerate(per_rank):
            assert np.array_equal(O, O0) and np.array_equal(L, L0), (it, r)   # bitwise across ranks
        gate(O0, L0, O_ref, L_ref, what=f"fused P={world} {schedule} launch {it}")
    assert all(np.array_equal(outs[0][0][0], o[0][0]) for o in outs)          # deterministic over launches


@pytest.mark.parametrize("world", [2, 3, 8])
def test_fused_exchange_gqa_and_ragged(world):
    p = synth.Problem(3, 16, 2, 128, [700, 4096, 2049], dtype="bf16", dist="D1", seed=72)
    O_ref, L_ref = run_oracle(p)
    for per_rank in _run_fused(p, world, launches=2):
        for O, L in per_rank:
            gate(O, L, O_ref, L_ref, what=f"fused GQA P={world}")


@pytest.mark.parametrize("group", [1, 8])
def test_fused_exchange_fp8(group):
    """FP8 KV shards (NEXT-4) through the fused exchange: v_scale is applied before the push."""
    p = synth.Problem(2, 2 * group, 2, 128, [3000, 5333], dtype="fp8", dist="D2", seed=74)
    O_ref, L_ref = run_oracle(p)
    for per_rank in _run_fused(p, 4, launches=2):
        O0, L0 = per_rank[0]
        for O, L in per_rank:
            assert np.array_equal(O, O0) and np.array_equal(L, L0)
        gate(O0, L0, O_ref, L_ref, what=f"fused fp8 g{group}")


def test_fused_exchange_multi_token_full():
    p = synth.Problem(2, 4, 2, 64, [999, 2500], dtype="fp16", dist="D1", seed=73, q_len=2)
    O_ref, L_ref = run_oracle(p, causal=False)
    for O, L in _run_fused(p, 2, launches=2, causal=False)[-1]:
        gate(O, L, O_ref, L_ref, what="fused N_q=2 non-causal")


def test_fused_exchange_requires_peers():
    import paper_2405_10480_b200 as la
    p = synth.Problem(1, 2, 2, 64, [256], dtype="bf16")
    plan = la.Plan(1, 2, 2, 64, [128], xchg_world=2, xchg_rank=0)
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda", token_range=[(0, 128)])
    with pytest.raises(la.LaError) as e:
        plan.decode(q, k, k)
    assert e.value.status == la.LA_ERR_STATE
    assert len(plan.xchg_handle()) == 64


def test_fused_exchange_timeout_is_reported():
    """A rank whose peer never launches gives up after 5 s and reports LA_ERR_TIMEOUT
    (instead of hanging the GPU)."""
    import paper_2405_10480_b200 as la
    p = synth.Problem(1, 1, 1, 64, [512], dtype="bf16")
    plans = [la.Plan(1, 1, 1, 64, [256], xchg_world=2, xchg_rank=r, grid=2) for r in range(2)]
    plans[0].xchg_attach(1, plans[1])
    plans[1].xchg_attach(0, plans[0])
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda", token_range=[(0, 256)])
    plans[0].decode(q, k, k)          # rank 1 never runs
    with pytest.raises(la.LaError) as e:
        plans[0].xchg_status()
    assert e.value.status == la.LA_ERR_TIMEOUT
