"""Producer-warp accounting (DESIGN §6 "Paged pools"): on a -DLA_PROF build the trace carries the
producer's cycles waiting for free ring slots and (paged) inside produce_paged.

  NAME=prof bash scripts/build_variant.sh wt -DLA_PROF
  LEANATTN_LIB=paper_2405_10480_b200/lib/variants/prof.so python scripts/producer_profile.py
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, synth, paper_2405_10480_b200 as la
for cfg, ps, eng in (("c3", 16, "mma"), ("c3", 0, "mma"), ("c2", 16, "auto"), ("c2", 0, "auto")):
    if ps:
        p = synth.config(cfg, layout="paged", page_size=ps)
        bt, num_pages = synth.paged_meta(p)
        k = torch.randn(num_pages, p.heads_kv, ps, p.head_dim, device="cuda").to(torch.bfloat16)
        kw = dict(layout="paged", block_table=bt, page_size=ps, num_pages=num_pages)
    else:
        p = synth.config(cfg)
        k = torch.randn(p.batch, p.heads_kv, p.max_ctx, p.head_dim, device="cuda").to(torch.bfloat16)
        kw = {}
    v = torch.randn_like(k)
    q = torch.randn(p.batch, p.heads_q, p.head_dim, device="cuda").to(torch.bfloat16)
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, engine=eng, schedule="streamk", trace=True, **kw)
    for _ in range(5): plan.decode(q, k, v)
    torch.cuda.synchronize()
    tr = plan.trace().astype(np.int64)
    span = (tr[:, 5] - tr[:, 1]) / 1e3
    pw, wait, work, n = tr[:, 0], tr[:, 2], tr[:, 3], tr[:, 4]
    cyc = span * 1.965e3
    print(f"{cfg} page {ps} {eng}: span med {np.median(span):.1f} us; producer slot-wait fraction {np.median(pw / cyc):.2f}; "
          f"consumer w0 wait frac {np.median(wait / cyc):.2f} work frac {np.median(work / cyc):.2f} stages {np.median(n):.0f}; produce_paged frac {np.median(tr[:, 6] / cyc):.2f}")
    del k, v; torch.cuda.empty_cache()
