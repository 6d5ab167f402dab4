"""Small decodes for compute-sanitizer (memcheck / racecheck / synccheck): MHA + GQA (mma.sync
and tcgen05 engines) + FP8, static and dynamic schedules, ragged tails, forced grids (the flag /
fold protocols)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402

for p, grid, tile, engine in ((synth.Problem(2, 2, 2, 128, [700, 333], dist="D2", seed=5), 5, 64, "mma"),
                              (synth.Problem(2, 8, 2, 128, [700, 333], dist="D2", seed=6), 4, 64, "mma"),
                              (synth.Problem(2, 8, 2, 128, [700, 333], dist="D2", seed=6), 4, 128, "tcgen05"),
                              (synth.Problem(2, 8, 2, 128, [700, 333], dtype="fp8", dist="D2", seed=8), 4, 128, "mma"),
                              (synth.Problem(1, 1, 1, 64, [4096], dtype="fp32", dist="D1", seed=7), 0, 0, "mma")):
    if len(sys.argv) > 1 and engine != sys.argv[1]:
        continue
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    for sched in ("streamk", "dynamic"):
        plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, grid=grid,
                       tile_n=tile, schedule=sched, engine=engine,
                       **(dict(k_scale=p.k_scale, v_scale=p.v_scale) if p.dtype == "fp8" else {}))
        for _ in range(2):
            out, lse = plan.decode(q, k, v)
        torch.cuda.synchronize()
        assert torch.isfinite(out).all()
# r02 paths: tcgen05 16 / 32-row tiles (deferred PV wait, wide epilogue staging the idle ring),
# paged pools on every engine (lane-distributed block-table window, elected loads), weighted
# stream-K ranges
extra = [(synth.Problem(2, 8, 2, 128, [900, 333], dist="D2", seed=9, q_len=2), 5, 128, "tcgen05", {}),
         (synth.Problem(2, 8, 2, 128, [900, 333], dist="D2", seed=9, q_len=4), 5, 128, "tcgen05", {}),
         (synth.Problem(1, 8, 1, 128, [3000], dist="D2", seed=10, q_len=4), 0, 32, "tcgen05", {})]
for eng, g in (("mma", 1), ("mma", 8), ("tcgen05", 8)):
    pp = synth.Problem(2, 2 * g, 2, 128, [700, 333], dist="D2", seed=11, layout="paged", page_size=16)
    bt, n = synth.paged_meta(pp)
    extra.append((pp, 5, 64, eng, dict(block_table=bt, page_size=16, num_pages=n)))
pf = synth.Problem(2, 8, 2, 128, [700, 333], dtype="fp8", dist="D2", seed=12, layout="paged", page_size=16)
bt, n = synth.paged_meta(pf)
extra.append((pf, 5, 128, "mma", dict(block_table=bt, page_size=16, num_pages=n, k_scale=pf.k_scale, v_scale=pf.v_scale)))
for p, grid, tile, engine, kw in extra:
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, grid=grid, tile_n=tile,
                   schedule="streamk", engine=engine, layout=p.layout, q_len=p.q_len, **kw)
    for weights in (None, [1 + (7 * i) % 13 for i in range(plan.info.grid)]):
        plan.set_weights(weights)
        for _ in range(2):
            out, lse = plan.decode(q, k, v)
        torch.cuda.synchronize()
        assert torch.isfinite(out).all()
print("sanitize case ok")
