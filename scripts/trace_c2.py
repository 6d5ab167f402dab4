"""Per-CTA timeline of a decode (la_plan_trace): SM-balance evidence (the paper's E2
occupancy analog).  Prints a summary and writes gpurun_out/trace_<cfg>_<sched>.csv.

  python scripts/trace_c2.py [c2|c3|c4] [dynamic|streamk]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402


def main(cfg="c2", schedule="dynamic", reps=5):
    p = synth.config(cfg)
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, layout=p.layout,
                   trace=True, schedule=schedule)
    for _ in range(3):
        plan.decode(q, k, v)
    for r in range(reps):
        torch.cuda.synchronize()
        plan.decode(q, k, v)
        tr = plan.trace().astype(np.int64)
    t0 = tr[:, 1].min()
    start = (tr[:, 1] - t0) / 1e3
    end = (tr[:, 5] - t0) / 1e3
    wait = np.where(tr[:, 3] > 0, (tr[:, 4] - tr[:, 3]) / 1e3, 0.0)
    dur = end - start
    smid = tr[:, 0]
    summary = dict(cfg=cfg, schedule=schedule, ctas=len(tr), vctas=int(plan.info.num_vctas),
                   kernel_us=float(end.max()), end_min_us=float(end.min()), end_med_us=float(np.median(end)),
                   idle_frac=float(1 - dur.mean() / end.max()), wait_max_us=float(wait.max()))
    line = json.dumps(summary)
    if schedule == "streamk":  # static: per-CTA work is known -> per-CTA bandwidth
        rows = plan.export()
        iters = np.bincount(rows[:, 0], weights=rows[:, 3] - rows[:, 2], minlength=len(tr))
        gbs = iters * 2 * plan.info.tile_n * p.head_dim * 2 / (dur * 1e-6) / 1e9
        print(line)
        print("per-CTA GB/s: min %.1f med %.1f max %.1f" % (gbs.min(), np.median(gbs), gbs.max()))
    else:
        print(line)
        claims, tiles = tr[:, 3], tr[:, 4]
        order = np.argsort(end)[::-1][:6]
        for g in order:
            print(f"cta {g} smid {smid[g]} end {end[g]:.1f} us claims {claims[g]} tiles {tiles[g]} "
                  f"GB/s {tiles[g] * 2 * plan.info.tile_n * p.head_dim * 2 / (dur[g] * 1e-6) / 1e9:.1f}")
        print("tiles per CTA: min %d med %d max %d" % (tiles.min(), np.median(tiles), tiles.max()))
        wait = np.zeros_like(end)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/trace_{cfg}_{schedule}.csv", "w") as f:
        f.write("cta,smid,start_us,wait_us,end_us\n")
        for g in range(len(tr)):
            f.write(f"{g},{smid[g]},{start[g]:.3f},{wait[g]:.3f},{end[g]:.3f}\n")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "c2", sys.argv[2] if len(sys.argv) > 2 else "dynamic")
