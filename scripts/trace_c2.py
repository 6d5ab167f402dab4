"""Per-CTA timeline of the c2 decode (la_plan_trace): SM-balance evidence (the paper's E2
occupancy analog).  Prints a summary and writes gpurun_out/trace_<cfg>.csv."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402


def main(cfg="c2", reps=5, **plan_kw):
    p = synth.config(cfg)
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, layout=p.layout,
                   trace=True, **plan_kw)
    for _ in range(3):
        plan.decode(q, k, v)
    res = []
    for r in range(reps):
        torch.cuda.synchronize()
        plan.decode(q, k, v)
        tr = plan.trace().astype(np.int64)
        t0 = tr[:, 1].min()
        start = (tr[:, 1] - t0) / 1e3
        end = (tr[:, 5] - t0) / 1e3
        wait = np.where(tr[:, 3] > 0, (tr[:, 4] - tr[:, 3]) / 1e3, 0.0)
        pub = np.where(tr[:, 2] > 0, (tr[:, 2] - t0) / 1e3, np.nan)
        dur = end - start
        res.append(dict(rep=r, kernel_us=float(end.max()), start_spread_us=float(start.max()),
                        end_min_us=float(end.min()), end_med_us=float(np.median(end)),
                        dur_min=float(dur.min()), dur_med=float(np.median(dur)), dur_max=float(dur.max()),
                        wait_max_us=float(wait.max()), wait_mean_us=float(wait.mean())))
    print(json.dumps(res[-1]))
    smid = tr[:, 0]
    order = np.argsort(smid)
    # work per CTA (iterations) and per-CTA bandwidth
    rows = plan.export()
    iters = np.bincount(rows[:, 0], weights=rows[:, 3] - rows[:, 2], minlength=len(tr))
    bytes_per_iter = 2 * plan.info.tile_n * p.head_dim * 2
    gbs = iters * bytes_per_iter / (dur * 1e-6) / 1e9
    print("per-CTA GB/s: min %.1f med %.1f max %.1f" % (gbs.min(), np.median(gbs), gbs.max()))
    # split by smid halves (die proxy) and by TPC parity
    for name, mask in (("smid<74", smid < 74), ("smid>=74", smid >= 74), ("even", smid % 2 == 0), ("odd", smid % 2 == 1)):
        if mask.any():
            print(f"{name:9s} n={mask.sum():3d} GB/s mean {gbs[mask].mean():.1f} dur mean {dur[mask].mean():.1f} us")
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/trace_{cfg}.csv", "w") as f:
        f.write("cta,smid,start_us,publish_us,wait_us,end_us,iters,gbs\n")
        for g in range(len(tr)):
            f.write(f"{g},{smid[g]},{start[g]:.3f},{pub[g]:.3f},{wait[g]:.3f},{end[g]:.3f},{int(iters[g])},{gbs[g]:.1f}\n")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["c2"]))
