"""Launch overhead study: event-timed kernel time vs the traced CTA span (la_plan_trace),
for a few configs (the cooperative-vs-plain comparison in DESIGN.md §6 used a temporary
LA_EXPERIMENT_NONCOOP switch in launch_decode, since removed).

  python scripts/launch_overhead.py c1 c3:fp8 c2 c3:tcgen05
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402


def case(spec):
    cfg, _, dt = spec.partition(":")
    engine = "mma"
    if dt == "tcgen05":
        dt, engine = "", "tcgen05"
    p = synth.config(cfg, **({"dtype": dt} if dt else {}))
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    kw = dict(k_scale=p.k_scale, v_scale=p.v_scale) if p.dtype == "fp8" else {}
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, trace=True, engine=engine, **kw)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ks, spans, starts = [], [], []
    for r in range(60):
        flush.zero_()
        e0.record()
        plan.decode(q, k, v)
        e1.record()
        torch.cuda.synchronize()
        tr = plan.trace().astype(np.int64)
        if r >= 10:
            ks.append(e0.elapsed_time(e1) * 1e3)
            spans.append((tr[:, 5].max() - tr[:, 1].min()) / 1e3)
            starts.append((tr[:, 1].max() - tr[:, 1].min()) / 1e3)
    coop = "coop"
    print(f"{spec:8s} {coop:5s} kernel_us med {np.median(ks):8.2f}  traced span {np.median(spans):8.2f}  "
          f"overhead {np.median(ks) - np.median(spans):6.2f}  CTA start spread {np.median(starts):5.2f}", flush=True)


if __name__ == "__main__":
    for s in sys.argv[1:]:
        case(s)
