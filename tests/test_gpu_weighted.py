"""GPU parity of the SM-rate-weighted stream-K schedule (la_plan_set_weights /
la_plan_calibrate): any contiguous ranges give Eq. 1 exactly, so the
weighted plans are gated against the fp64 oracle like every other schedule, they are bitwise
reproducible for fixed weights, a captured CUDA graph replays them, and calibration leaves
a correct, weighted plan."""
import numpy as np
import pytest
import torch

import synth
from _helpers import cuda_inputs, gate, run_oracle, oracle_unit

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as la
    la.lib()


def _plan(la, p, **kw):
    return la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, layout=p.layout,
                   max_ctx=p.max_ctx if p.layout == "bhsd" else 0, schedule="streamk",
                   **(dict(q_len=p.q_len) if p.q_len > 1 else {}), **kw)


@pytest.mark.parametrize("group,q_len,engine", [(1, 1, "auto"), (8, 1, "mma"), (8, 1, "tcgen05"),
                                                (8, 2, "tcgen05"), (8, 4, "tcgen05")])
def test_random_weights_parity_and_determinism(group, q_len, engine):
    import paper_2405_10480_b200 as la
    p = synth.Problem(3, 2 * group, 2, 128, [3000, 517, 2048], dtype="bf16", dist="D2", seed=71, q_len=q_len)
    O_ref, L_ref = run_oracle(p)
    q, k, v = cuda_inputs(p)
    rng = np.random.default_rng(group * 10 + q_len)
    for grid, tile_n in ((0, 64), (7, 32), (37, 128)):
        plan = _plan(la, p, grid=grid, tile_n=tile_n, engine=engine)
        G = plan.info.grid
        for w in (rng.integers(1, 1 << 20, size=G), rng.integers(60000, 70000, size=G), np.full(G, 3)):
            plan.set_weights(w)
            out, lse = plan.decode(q, k, v)
            torch.cuda.synchronize()
            plan.status()
            gate(out.cpu().numpy(), lse.cpu().numpy(), O_ref, L_ref, what=f"weighted g{group} Nq{q_len} G{grid} T{tile_n}")
            ref = out.clone()
            for _ in range(3):
                assert torch.equal(plan.decode(q, k, v)[0], ref)


def test_graph_replays_after_set_weights():
    import paper_2405_10480_b200 as la
    p = synth.Problem(2, 16, 2, 128, [5000, 1200], dtype="bf16", dist="D1", seed=72)
    q, k, v = cuda_inputs(p)
    plan = _plan(la, p, engine="mma")
    out = torch.empty(2, 16, 128, dtype=torch.float32, device="cuda")
    lse = torch.empty(2, 16, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.decode(q, k, v, out, lse, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.decode(q, k, v, out, lse, stream=s)
    G = plan.info.grid
    rng = np.random.default_rng(9)
    for trial in range(3):
        plan.set_weights(rng.integers(1000, 5000, size=G), stream=s)
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        eager = plan.decode(q, k, v)[0]
        torch.cuda.synchronize()
        assert torch.equal(out, eager), trial


@pytest.mark.parametrize("cfg,engine", [("c3", "mma"), ("c3", "tcgen05")])
def test_calibrate_full_size(cfg, engine):
    """la_plan_calibrate at BASELINE size (the bench's launch configuration): the plan ends
    weighted, within one LeanTile of rate-proportional, and still matches the oracle."""
    import paper_2405_10480_b200 as la
    p = synth.config(cfg)
    q, k, v = cuda_inputs(p)
    plan = _plan(la, p, engine=engine)
    rl = plan.calibrate(q, k, v, launches=3, rounds=2)
    assert plan.info.sm_weighted == 1 and rl.sum() == plan.info.total_iters and rl.min() >= 1
    plan.status()
    out, lse = plan.decode(q, k, v)
    torch.cuda.synchronize()
    O, L = out.cpu().numpy(), lse.cpu().numpy()
    for b, h in ((0, 0), (5, 3), (7, 7)):
        O_ref, L_ref = oracle_unit(p, b, h)
        gate(O[b, 8 * h:8 * h + 8], L[b, 8 * h:8 * h + 8], O_ref, L_ref, what=f"{cfg} calibrated b{b} h{h}")
    plan.set_weights(None)
    assert plan.info.sm_weighted == 0 and plan.range_lengths().max() - plan.range_lengths().min() <= 1


def test_calibrate_rejects_dynamic_and_exchange_plans():
    import paper_2405_10480_b200 as la
    p = synth.Problem(1, 4, 4, 128, [5000], dtype="bf16", dist="D1", seed=73)
    q, k, v = cuda_inputs(p)
    for kw in (dict(schedule="dynamic"), dict(schedule="streamk", xchg_world=2, xchg_rank=0)):
        plan = la.Plan(1, 4, 4, 128, [5000], **kw)
        with pytest.raises(la.LaError) as e:
            plan.calibrate(q, k, v, launches=1, rounds=1)
        assert e.value.status == la.LA_ERR_STATE, kw
    plan = la.Plan(1, 4, 4, 128, [5000], schedule="streamk")
    with pytest.raises(la.LaError) as e:
        plan.calibrate(q, k, v, launches=0, rounds=1)
    assert e.value.status == la.LA_ERR_INVALID


@pytest.mark.parametrize("layout,dtype", [("paged", "bf16"), ("bhsd", "fp8"), ("packed", "bf16")])
def test_random_weights_other_layouts(layout, dtype):
    """Weighted ranges on a paged pool (tcgen05 engine under AUTO), an FP8 cache and a packed
    ragged cache: oracle-gated and bitwise reproducible."""
    import paper_2405_10480_b200 as la
    kw = dict(page_size=16) if layout == "paged" else {}
    p = synth.Problem(3, 16, 2, 128, [3000, 517, 2048], dtype=dtype, dist="D2", seed=74, layout=layout, **kw)
    O_ref, L_ref = run_oracle(p)
    q, k, v = cuda_inputs(p)
    extra = {}
    if layout == "paged":
        bt, num_pages = synth.paged_meta(p)
        extra = dict(block_table=bt, page_size=16, num_pages=num_pages)
    if dtype == "fp8":
        extra.update(k_scale=p.k_scale, v_scale=p.v_scale)
    rng = np.random.default_rng(11)
    for grid, tile_n in ((0, 64), (9, 128)):
        plan = _plan(la, p, grid=grid, tile_n=tile_n, **extra)
        plan.set_weights(rng.integers(1, 1 << 20, size=plan.info.grid))
        out, lse = plan.decode(q, k, v)
        torch.cuda.synchronize()
        plan.status()
        gate(out.cpu().numpy(), lse.cpu().numpy(), O_ref, L_ref, what=f"weighted {layout}/{dtype} G{grid} T{tile_n}")
        ref = out.clone()
        assert torch.equal(plan.decode(q, k, v)[0], ref)
