"""Per-CTA timeline of one decode launch for latency analysis (la_plan_trace), plus the
event-timed kernel duration, so launch overhead = kernel_us - traced span.

  python scripts/trace_case.py c1 streamk 256
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402


def main(cfg, schedule, tile_n, flush_mode="write"):
    p = synth.config(cfg)
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, layout=p.layout,
                   trace=True, schedule=schedule, tile_n=tile_n)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ks = []
    for r in range(20):
        if flush_mode == "write":
            flush.zero_()
        elif flush_mode == "read":
            flush.sum()
        e0.record()
        plan.decode(q, k, v)
        e1.record()
        torch.cuda.synchronize()
        ks.append(e0.elapsed_time(e1) * 1e3)
    tr = plan.trace().astype(np.int64)
    t0 = tr[:, 1].min()
    rel = lambda c: np.where(tr[:, c] > 0, (tr[:, c] - t0) / 1e3, np.nan)
    print(f"[flush {flush_mode}] {cfg} {schedule} tile {plan.info.tile_n} grid {plan.info.grid} vctas {plan.info.num_vctas} "
          f"kernel_us med {np.median(ks):.2f} traced span {rel(5).max():.2f}")
    print(" cta smid  start  publish  wait0  wait1   end")
    for g in range(len(tr)):
        print(f"{g:4d} {tr[g, 0]:4d} {rel(1)[g]:6.2f} {rel(2)[g]:7.2f} {rel(3)[g]:6.2f} {rel(4)[g]:6.2f} {rel(5)[g]:6.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), *(sys.argv[4:5]))
