"""la_decode captured into a CUDA graph (the serving pattern: one capture, many replays with
new cache contents in the same buffers).  The flag epoch of Alg. 2's Signal/Wait lives on the
device (reading C17), so every replay publishes fresh flags: each replay must equal an eager
decode of the same inputs bit for bit, and the oracle within the parity gates."""
import numpy as np
import pytest
import torch

import synth
from _helpers import gate, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as la
    la.lib()


CASES = [  # (problem args, grid, tile_n, schedule, engine): peers must be waited on (grid > units)
    (dict(batch=2, heads_q=4, heads_kv=4, head_dim=128, ctx_lens=[3000, 777]), 9, 64, "streamk", "mma"),
    (dict(batch=2, heads_q=16, heads_kv=2, head_dim=128, ctx_lens=[3000, 777]), 7, 128, "streamk", "mma"),
    (dict(batch=2, heads_q=16, heads_kv=2, head_dim=128, ctx_lens=[3000, 777]), 7, 128, "streamk", "tcgen05"),
    (dict(batch=2, heads_q=16, heads_kv=2, head_dim=128, ctx_lens=[3000, 777]), 7, 64, "dynamic", "mma"),
]


@pytest.mark.parametrize("args,grid,tile_n,schedule,engine", CASES)
def test_graph_replay_matches_eager_and_oracle(args, grid, tile_n, schedule, engine):
    import paper_2405_10480_b200 as la
    problems = [synth.Problem(**args, dtype="bf16", dist="D2", seed=100 + i) for i in range(3)]
    p0 = problems[0]
    q = synth.gen_q(p0, "cuda")
    k = synth.fill_kv_cache(p0, "k", "cuda")
    v = synth.fill_kv_cache(p0, "v", "cuda")
    kw = dict(grid=grid, tile_n=tile_n, schedule=schedule, engine=engine)
    plan = la.Plan(p0.batch, p0.heads_q, p0.heads_kv, p0.head_dim, p0.ctx_lens, **kw)
    out = torch.empty(p0.batch, p0.heads_q, p0.head_dim, dtype=torch.float32, device="cuda")
    lse = torch.empty(p0.batch, p0.heads_q, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        plan.decode(q, k, v, out, lse, stream=s)  # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.decode(q, k, v, out, lse, stream=s)
    eager = la.Plan(p0.batch, p0.heads_q, p0.heads_kv, p0.head_dim, p0.ctx_lens, **kw)
    for rep in range(2):
        for p in problems:  # new contents in the captured buffers, then replay
            q.copy_(synth.gen_q(p, "cuda"))
            k.copy_(synth.fill_kv_cache(p, "k", "cuda"))
            v.copy_(synth.fill_kv_cache(p, "v", "cuda"))
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            ref_o, ref_l = eager.decode(q, k, v)
            torch.cuda.synchronize()
            assert torch.equal(out, ref_o) and torch.equal(lse, ref_l), f"replay {rep} seed {p.seed}"
            if rep == 0:
                O_ref, L_ref = run_oracle(p)
                gate(out.cpu().numpy().astype(np.float64), lse.cpu().numpy().astype(np.float64), O_ref, L_ref,
                     what=f"graph {engine}/{schedule} seed {p.seed}")
