"""Serving-loop cost of per-step re-planning (la_plan_update): c4 (16 ragged requests,
1k-128k tokens, 32 heads) decoded K steps with every context length growing by one token per
step, vs the same K decodes on a fixed plan -- CUDA events over the whole loop (the update's
host work and its one async upload are inside the timed region), plus the same loop replayed
from ONE captured CUDA graph (updates between replays).

  python scripts/update_loop.py [--steps K] [--config c4]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=50)
ap.add_argument("--config", default="c4")
a = ap.parse_args()
p0 = synth.config(a.config)
cap = max(p0.ctx_lens) + a.steps + 1
p = synth.Problem(p0.batch, p0.heads_q, p0.heads_kv, p0.head_dim, p0.ctx_lens, dtype=p0.dtype, seed=p0.seed,
                  max_ctx=cap)
q = synth.gen_q(p, "cuda")
k = synth.fill_kv_cache(p, "k", "cuda")   # capacity-sized BHSD caches (rows past n_b are zero)
v = synth.fill_kv_cache(p, "v", "cuda")
s = torch.cuda.Stream()          # a non-default stream (CUDA graph capture needs one)
s.wait_stream(torch.cuda.current_stream())
torch.cuda.set_stream(s)
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, max_ctx=cap)
out = torch.empty(p.batch, p.heads_q, p.head_dim, dtype=torch.float32, device="cuda")
lse = torch.empty(p.batch, p.heads_q, dtype=torch.float32, device="cuda")


def timed(fn):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for i in range(a.steps):
        fn(i)
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / a.steps


def decode_only(i):
    plan.decode(q, k, v, out, lse, stream=s)


def update_and_decode(i):
    plan.update([n + i for n in p.ctx_lens], stream=s)
    plan.decode(q, k, v, out, lse, stream=s)


base = timed(decode_only)
upd = timed(update_and_decode)
# one CUDA graph, captured once, replayed after every update
plan.update(p.ctx_lens, stream=s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    plan.decode(q, k, v, out, lse, stream=s)


def graph_step(i):
    plan.update([n + i for n in p.ctx_lens], stream=s)
    g.replay()


grp = timed(graph_step)
plan.status()
print(json.dumps({"config": a.config, "steps": a.steps, "schedule": la.leanattn.SCHEDULE_NAMES[plan.info.schedule],
                  "decode_only_us": base, "update_plus_decode_us": upd, "overhead_pct": 100 * (upd / base - 1),
                  "graph_replay_after_update_us": grp, "graph_overhead_pct": 100 * (grp / base - 1),
                  "updates": plan.info.updates}))
