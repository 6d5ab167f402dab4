"""Which CTAs end late and why: per-CTA (start, publish, host-wait begin/end, end) from
la_plan_trace (normal build), for one engine.   python scripts/trace_tail.py c3 tcgen05"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402

cfg, engine = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "mma")
p = synth.config(cfg)
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, trace=True, engine=engine)
for _ in range(5):
    plan.decode(q, k, v)
torch.cuda.synchronize()
tr = plan.trace().astype(np.int64)
t0 = tr[:, 1].min()
rel = lambda c: np.where(tr[:, c] > 0, (tr[:, c] - t0) / 1e3, np.nan)
st, pub, w0, w1, en = rel(1), rel(2), rel(3), rel(4), rel(5)
print(f"{cfg} {engine}: end us min/med/max {np.nanmin(en):.1f}/{np.nanmedian(en):.1f}/{np.nanmax(en):.1f}  start max {np.nanmax(st):.1f}")
seg = plan.export()
for g in np.argsort(en)[-8:]:
    print(f"  CTA {g}: start {st[g]:.1f} publish {pub[g]:.1f} wait {w0[g]:.1f}->{w1[g]:.1f} end {en[g]:.1f} segs {seg[seg[:, 0] == g].tolist()}")
for g in np.argsort(en)[:3]:
    print(f"  fast CTA {g}: start {st[g]:.1f} publish {pub[g]:.1f} wait {w0[g]:.1f}->{w1[g]:.1f} end {en[g]:.1f}")
