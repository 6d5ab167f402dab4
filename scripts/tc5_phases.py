"""Cycles per 128-token stage of one tcgen05 warpgroup, by phase (DESIGN §6 tcgen05 round-2
changes): needs a -DLA_TC5_PROF build, which prints one line per sampled CTA / warpgroup.

  NAME=tc5prof bash scripts/build_variant.sh wt -DLA_TC5_PROF
  LEANATTN_LIB=paper_2405_10480_b200/lib/variants/tc5prof.so python scripts/tc5_phases.py
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch, synth, paper_2405_10480_b200 as la
for ql, eng in ((4, "tcgen05"), (2, "tcgen05"), (1, "tcgen05")):
    p = synth.config("c3", **(dict(q_len=ql) if ql > 1 else {}))
    q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, q_len=ql, engine=eng)
    for _ in range(2): plan.decode(q, k, v)
    torch.cuda.synchronize()
    print("----", flush=True)
    del q, k, v; torch.cuda.empty_cache()
