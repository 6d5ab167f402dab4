"""Paged pools vs block-table order and engine (DESIGN §6 "Paged pools"): c2 / c3 at page 16 / 64 /
256 with the seeded random block table and a sequential one, mma.sync and tcgen05 for GQA.

  python scripts/paged_engines.py c3
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, synth, paper_2405_10480_b200 as la
cfg = sys.argv[1]
for ps in (16, 64, 256):
    p = synth.config(cfg, layout="paged", page_size=ps)
    bt, num_pages = synth.paged_meta(p)
    need = [-(-n // ps) for n in p.ctx_lens]
    ident = np.full_like(bt, num_pages - 1)
    pos = 0
    for b, k in enumerate(need):
        ident[b, :k] = np.arange(pos, pos + k); pos += k
    k = torch.randn(num_pages, p.heads_kv, ps, p.head_dim, device="cuda").to(torch.bfloat16)
    v = torch.randn_like(k)
    q = torch.randn(p.batch, p.heads_q, p.head_dim, device="cuda").to(torch.bfloat16)
    for name, table in (("random", bt), ("sequential", ident)):
        for engine in (("mma", "tcgen05") if p.group > 1 else ("auto",)):
            plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, layout="paged", block_table=table,
                           page_size=ps, num_pages=num_pages, engine=engine)
            for _ in range(5): plan.decode(q, k, v)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(50): plan.decode(q, k, v)
            e1.record(); torch.cuda.synchronize()
            print(f"{cfg} page {ps:3d} {name:10s} {engine:7s} {e0.elapsed_time(e1) / 50 * 1e3:7.1f} us/step")
    del k, v
    torch.cuda.empty_cache()
