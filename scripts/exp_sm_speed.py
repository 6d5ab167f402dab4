"""Is per-SM streaming speed a stable property of the SM (static schedule, per-CTA trace)?
Correlates per-smid GB/s across launches and across configs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402


def per_sm(cfg, reps=6):
    p = synth.config(cfg)
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, trace=True)
    rows = plan.export()
    iters = np.bincount(rows[:, 0], weights=rows[:, 3] - rows[:, 2], minlength=plan.info.grid)
    out = []
    for r in range(reps + 2):
        torch.cuda.synchronize()
        plan.decode(q, k, v)
        tr = plan.trace().astype(np.int64)
        if r < 2:
            continue
        dur = (tr[:, 5] - tr[:, 1]) / 1e3
        gbs = iters * 2 * plan.info.tile_n * p.head_dim * 2 / (dur * 1e-6) / 1e9
        sm = np.full(148, np.nan)
        sm[tr[:, 0]] = gbs
        out.append(sm)
    return np.array(out)


for cfg in ("c2", "c3"):
    a = per_sm(cfg)
    c = np.corrcoef(a)
    off = c[~np.eye(len(a), dtype=bool)]
    print(cfg, "per-SM GB/s spread (min/med/max of run-mean):", np.round(np.nanmin(a.mean(0)), 1),
          np.round(np.nanmedian(a.mean(0)), 1), np.round(np.nanmax(a.mean(0)), 1),
          "| run-to-run corr of per-SM speed: min %.2f mean %.2f" % (off.min(), off.mean()))
    if cfg == "c2":
        a2 = a
    else:
        print("c2 vs c3 per-SM speed corr: %.2f" % np.corrcoef(a2.mean(0), a.mean(0))[0, 1])
        np.save("gpurun_out/sm_speed.npy", np.stack([a2.mean(0), a.mean(0)]))
