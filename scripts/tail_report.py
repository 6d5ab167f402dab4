"""Where the time between launch and the last CTA goes: per-CTA timeline (la_plan_trace) of
one workload under one schedule / engine, next to the CUDA-event kernel time.

  python scripts/tail_report.py CFG [--schedule S] [--engine E] [--first F] [--min M] [--q-len N]

Prints: event-timed kernel µs (median of 20), the traced span (first CTA start -> last CTA
end), CTA start / end spread, per-CTA streaming rate spread (KV bytes of the CTA's ranges /
its busy time), and the 5 latest CTAs.  SM balance analog of P:191 (ncu sm__cycles_active).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--schedule", default="streamk")
ap.add_argument("--engine", default="auto")
ap.add_argument("--first", type=int, default=940)
ap.add_argument("--min", type=int, default=2)
ap.add_argument("--q-len", type=int, default=1)
ap.add_argument("--dtype", default=None)
a = ap.parse_args()
kw = {"dtype": a.dtype} if a.dtype else {}
if a.q_len > 1:
    kw["q_len"] = a.q_len
p = synth.config(a.cfg, **kw)
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
fp8 = dict(k_scale=p.k_scale, v_scale=p.v_scale) if p.dtype == "fp8" else {}
common = dict(dtype=p.dtype, engine=a.engine, schedule=a.schedule, dyn_first_permille=a.first, dyn_min_chunk=a.min,
              q_len=a.q_len, **fp8)
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, **common)
tplan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, trace=True, **common)
s = torch.cuda.current_stream()
ts = []
for i in range(25):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    plan.decode(q, k, v)
    e1.record(s)
    torch.cuda.synchronize()
    if i >= 5:
        ts.append(e0.elapsed_time(e1) * 1e3)
for _ in range(3):
    tplan.decode(q, k, v)
torch.cuda.synchronize()
tr = tplan.trace().astype(np.int64)
t0 = tr[:, 1].min()
st = (tr[:, 1] - t0) / 1e3
en = (tr[:, 5] - t0) / 1e3
inf = plan.info
seg = plan.export()
tile_bytes = 2 * inf.tile_n * inf.head_dim * {"bf16": 2, "fp16": 2, "fp32": 4, "fp8": 1}[p.dtype]
print(f"{a.cfg} {a.schedule} engine={inf.engine} grid={inf.grid} vctas={inf.num_vctas} QE={inf.quantization_efficiency:.4f}")
print(f"  event kernel us: median {np.median(ts):.1f}  min {np.min(ts):.1f}  max {np.max(ts):.1f}")
print(f"  traced span {en.max():.1f} us; start max {st.max():.2f}; end min/p10/med/p90/max "
      f"{en.min():.1f}/{np.percentile(en, 10):.1f}/{np.median(en):.1f}/{np.percentile(en, 90):.1f}/{en.max():.1f}")
print(f"  mean CTA busy / span = {np.mean(en - st) / en.max():.4f}")
if a.schedule in ("streamk", "sequential"):
    iters = np.bincount(seg[:, 0], weights=seg[:, 3] - seg[:, 2], minlength=inf.grid)
    rate = iters * tile_bytes / np.maximum(en - st, 1e-3) / 1e3  # GB/s per CTA
    print(f"  per-CTA GB/s min/p10/med/p90/max {rate.min():.1f}/{np.percentile(rate, 10):.1f}/{np.median(rate):.1f}/"
          f"{np.percentile(rate, 90):.1f}/{rate.max():.1f}  (sum {rate.sum():.0f})")
    w = np.where(tr[:, 3] > 0, (tr[:, 4] - tr[:, 3]) / 1e3, 0)
    print(f"  host wait us: max {w.max():.2f}  mean(>0) {w[w > 0].mean() if (w > 0).any() else 0:.2f}")
else:
    print(f"  claims per CTA min/max {tr[:, 3].min()}/{tr[:, 3].max()}, LeanTiles per CTA min/max {tr[:, 4].min()}/{tr[:, 4].max()}")
    if os.environ.get("LA_EPI_TRACE"):  # a -DLA_EPI_TRACE build: fields 3, 4 are times (count-in done, fold done)
        ci = np.where(tr[:, 3] > 0, (tr[:, 3] - tr[:, 2]) / 1e3, np.nan)
        fo = np.where(tr[:, 4] > 0, (tr[:, 4] - tr[:, 3]) / 1e3, np.nan)
        print(f"  last segment -> count-in done: med {np.nanmedian(ci):.2f} p90 {np.nanpercentile(ci, 90):.2f} max {np.nanmax(ci):.2f} us;"
              f" fold: n {np.sum(~np.isnan(fo))} med {np.nanmedian(fo):.2f} max {np.nanmax(fo):.2f} us")
    lastseg = (tr[:, 2] - t0) / 1e3
    epi = en - lastseg
    print(f"  last segment taken by the epilogue: med {np.median(lastseg):.1f} max {lastseg.max():.1f}; "
          f"epilogue tail after it: med {np.median(epi):.2f} p90 {np.percentile(epi, 90):.2f} max {epi.max():.2f} us")
for g in np.argsort(en)[-5:]:
    extra = f" last seg {(tr[g, 2] - t0) / 1e3:.1f} claims {tr[g, 3]} tiles {tr[g, 4]}" if a.schedule in ("dynamic", "fixed_split") else ""
    print(f"  late CTA {g} smid {tr[g, 0]}: start {st[g]:.2f} end {en[g]:.1f}{extra}")
