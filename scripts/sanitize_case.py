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
print("sanitize case ok")
