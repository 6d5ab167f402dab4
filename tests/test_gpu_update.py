"""GPU parity of the per-step plan update (la_plan_update) and of the dynamic
schedule's fold tree on a shape whose counters collided in r01:

* update -> decode equals a fresh plan's decode of the same lengths bit for bit (same
  schedule) and the oracle within the parity gates, step after step, every layout;
* a CUDA graph captured once replays correctly after updates (nothing a launch takes by
  value depends on ctx_lens);
* the dynamic schedule on a colliding shape matches the oracle over repeated launches
  (a lost arrival would leave rows unwritten and the counters dirty for the next launch);
* la_plan_status reports no timeout after correct launches; fp32 at head_dim 128.
"""
import numpy as np
import pytest
import torch

import synth
from _helpers import cuda_inputs, gate, run_cuda, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as la
    la.lib()


def _np(t):
    return t.detach().cpu().numpy().astype(np.float64)


def test_dynamic_fold_tree_on_a_colliding_shape():
    """B = 3, 8 q-heads / 4 KV heads, lens [32544, 5404, 6961]: in the 148-CTA dynamic
    schedule a virtual CTA ends one unit's last fold group and hosts the next unit's first
    group (the r01 counter index collided there -- checked here on the plan's own export)."""
    import paper_2405_10480_b200 as la
    p = synth.Problem(3, 8, 4, 128, [32544, 5404, 6961], dtype="bf16", dist="D2", seed=31)
    q, k, v = cuda_inputs(p)
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, schedule="dynamic", engine="mma")
    # (r02 folds each unit by its last arriving piece; the shape stays as a regression case)
    O_ref, L_ref = run_oracle(p)
    first = None
    for it in range(4):   # counters must come back clean for every next launch
        o, l = plan.decode(q, k, v)
        torch.cuda.synchronize()
        gate(_np(o), _np(l), O_ref, L_ref, what=f"dynamic collide launch {it}")
        if first is None:
            first = (o.clone(), l.clone())
        else:
            assert torch.equal(o, first[0]) and torch.equal(l, first[1])
    plan.status()


def _layout_kw(p):
    if p.layout == "paged":
        bt, npages = synth.paged_meta(p)
        return dict(layout="paged", block_table=bt, page_size=p.page_size, num_pages=npages)
    return dict(layout=p.layout, max_ctx=p.max_ctx if p.layout == "bhsd" else 0)


STEPS = [[3000, 1, 2047], [3001, 2, 2048], [128, 700, 4096], [4096, 4096, 4096], [5, 3333, 64]]


@pytest.mark.parametrize("layout", ["bhsd", "paged"])
@pytest.mark.parametrize("heads,engine,schedule", [(4, "mma", "streamk"), (4, "mma", "dynamic"),
                                                    (16, "mma", "streamk"), (16, "tcgen05", "streamk"),
                                                    (8, "mma", "fixed_split")])
def test_update_loop_matches_fresh_plans_and_oracle(layout, heads, engine, schedule):
    """A serving loop: one plan, its lengths change every step (la_plan_update on the
    decode stream), the caches are the capacity-sized buffers of a D1 problem (element values
    do not depend on n_b), each step checked against a fresh plan and the oracle."""
    import paper_2405_10480_b200 as la
    cap = synth.Problem(3, heads, 2 if heads > 4 else 4, 128, [4096] * 3, dtype="bf16", dist="D1", seed=41,
                        layout=layout, page_size=64 if layout == "paged" else 0)
    q, k, v = cuda_inputs(cap)
    lkw = _layout_kw(cap)
    plan = la.Plan(cap.batch, cap.heads_q, cap.heads_kv, 128, STEPS[0], schedule=schedule, engine=engine, **lkw)
    launch = plan.info.grid
    for i, lens in enumerate(STEPS):
        plan.update(lens)
        o, l = plan.decode(q, k, v)
        torch.cuda.synchronize()
        assert plan.info.grid == launch and plan.info.updates == i + 1
        p = synth.Problem(3, cap.heads_q, cap.heads_kv, 128, lens, dtype="bf16", dist="D1", seed=41, layout=layout,
                          max_ctx=4096, page_size=cap.page_size)
        if layout == "paged":  # the capacity problem's pool and block table hold every step's tokens
            O_ref, L_ref = _oracle_paged_prefix(cap, lens)
        else:
            O_ref, L_ref = run_oracle(p)
        gate(_np(o), _np(l), O_ref, L_ref, what=f"{layout}/{engine}/{schedule} step {i}")
        fresh = la.Plan(cap.batch, cap.heads_q, cap.heads_kv, 128, lens, schedule=schedule, engine=engine,
                        grid=min(launch, plan.info.total_iters), **lkw)
        fo, fl = fresh.decode(q, k, v)
        torch.cuda.synchronize()
        assert np.array_equal(fresh.export(), plan.export())
        assert torch.equal(fo, o) and torch.equal(fl, l), f"step {i}: update != fresh plan"
    plan.status()


def _oracle_paged_prefix(cap, lens):
    """Oracle on the first lens[b] tokens of the capacity problem (D1: values independent of n)."""
    import oracle
    q = synth.to_f64(synth.gen_q(cap))
    outs, lses = [], []
    for b, n in enumerate(lens):
        ob, lb = [], []
        for h in range(cap.heads_kv):
            kk = synth.to_f64(synth.gen_kv_unit(cap, b, h, "k", "cpu", 0, n))
            vv = synth.to_f64(synth.gen_kv_unit(cap, b, h, "v", "cpu", 0, n))
            o, lse = oracle.decode_attention_unit(q[b, h * cap.group:(h + 1) * cap.group], kk, vv, cap.scale)
            ob.append(o)
            lb.append(lse)
        outs.append(np.concatenate(ob))
        lses.append(np.concatenate(lb))
    return np.stack(outs), np.stack(lses)


@pytest.mark.parametrize("heads,engine", [(4, "mma"), (16, "mma"), (16, "tcgen05"), (32, "tcgen05")])
def test_graph_replays_across_updates(heads, engine):
    """Capture la_decode once; update the lengths (on the capture stream) and replay: every
    replay equals an eager decode of a fresh plan for those lengths, bit for bit."""
    import paper_2405_10480_b200 as la
    cap = synth.Problem(2, heads, 2 if heads > 4 else 4, 128, [4096, 4096], dtype="bf16", dist="D1", seed=43)
    q, k, v = cuda_inputs(cap)
    plan = la.Plan(2, cap.heads_q, cap.heads_kv, 128, [1000, 4096], max_ctx=4096, engine=engine)
    out = torch.empty(2, cap.heads_q, 128, dtype=torch.float32, device="cuda")
    lse = torch.empty(2, cap.heads_q, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.decode(q, k, v, out, lse, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.decode(q, k, v, out, lse, stream=s)
    for lens in ([1000, 4096], [1001, 17], [4096, 4096], [1, 2], [2500, 3999]):
        plan.update(lens, stream=s)
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        fresh = la.Plan(2, cap.heads_q, cap.heads_kv, 128, lens, max_ctx=4096, engine=engine,
                        grid=plan.info.num_vctas)
        ro, rl = fresh.decode(q, k, v)
        torch.cuda.synchronize()
        assert torch.equal(out, ro) and torch.equal(lse, rl), lens
        p = synth.Problem(2, cap.heads_q, cap.heads_kv, 128, lens, dtype="bf16", dist="D1", seed=43, max_ctx=4096)
        O_ref, L_ref = run_oracle(p)
        gate(_np(out), _np(lse), O_ref, L_ref, what=f"graph after update {lens}")
    plan.status()


def test_async_initial_upload_on_a_stream():
    """la_plan with opts.stream: the table upload is left in flight on that stream; a decode
    on the same stream sees the tables."""
    import paper_2405_10480_b200 as la
    p = synth.Problem(2, 4, 4, 128, [3000, 777], dtype="bf16", dist="D2", seed=44)
    q, k, v = cuda_inputs(p)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan = la.Plan(2, 4, 4, 128, p.ctx_lens, stream=s, grid=11)
        o, l = plan.decode(q, k, v, stream=s)
    torch.cuda.synchronize()
    O_ref, L_ref = run_oracle(p)
    gate(_np(o), _np(l), O_ref, L_ref, what="async upload")


@pytest.mark.parametrize("dist", ["D1", "D2", "D4"])
def test_fp32_head_dim_128(dist):
    p = synth.Problem(2, 2, 2, 128, [3000, 1333], dtype="fp32", dist=dist, seed=45)
    O_ref, L_ref = run_oracle(p)
    inputs = cuda_inputs(p)
    for schedule in ("streamk", "dynamic"):
        for grid in (0, 7):
            O, L, plan = run_cuda(p, inputs=inputs, schedule=schedule, grid=grid)
            gate(O, L, O_ref, L_ref, what=f"fp32 d128 {dist} {schedule} G{grid}")


def test_binding_rejects_mismatched_tensors():
    import paper_2405_10480_b200 as la
    p = synth.Problem(1, 4, 4, 128, [1000], dtype="bf16", seed=46)
    q, k, v = cuda_inputs(p)
    plan = la.Plan(1, 4, 4, 128, p.ctx_lens)
    with pytest.raises(ValueError):
        plan.decode(q.float(), k, v)                       # wrong q dtype
    with pytest.raises(ValueError):
        plan.decode(q, k[:, :, :500].contiguous(), v)      # cache smaller than the plan's
    with pytest.raises(ValueError):
        plan.decode(q, k, v, out=torch.empty(1, 4, 64, device="cuda"))  # out too small
