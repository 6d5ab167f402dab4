"""Distribution of the traced kernel span over 40 launches (each the last of 3 back to back) and the
critical path of the slowest ones: the last CTA to end, its stream end, its wait on the peers' flags,
its fold (publish) and end (DESIGN §6 "Epilogue tail").

  PYTHONPATH=. python scripts/tail_dist.py Q_LEN [ENGINE]      e.g. 4 tcgen05
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, synth, paper_2405_10480_b200 as la
qlen = int(sys.argv[1]); eng = sys.argv[2] if len(sys.argv) > 2 else "tcgen05"
p = synth.config("c3", **(dict(q_len=qlen) if qlen > 1 else {}))
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, trace=True, engine=eng, schedule="streamk", q_len=qlen)
seg = plan.export()
rows = []
for rep in range(40):
    for _ in range(3): plan.decode(q, k, v)
    torch.cuda.synchronize()
    tr = plan.trace().astype(np.int64); t0 = tr[:, 1].min()
    rel = lambda x: np.where(x > 0, (x - t0) / 1e3, np.nan)
    st, pub, w0, w1, en, se = rel(tr[:, 1]), rel(tr[:, 2]), rel(tr[:, 3]), rel(tr[:, 4]), rel(tr[:, 5]), rel(tr[:, 6])
    g = int(np.nanargmax(en))
    rows.append((np.nanmax(en), np.nanmax(se), np.nanmedian(se), g, se[g], w0[g], w1[g], pub[g], en[g], np.nanmax(st)))
r = np.array(rows)
print(f"q{qlen} {eng}: span p10/p50/p90/max {np.percentile(r[:,0],10):.1f}/{np.median(r[:,0]):.1f}/{np.percentile(r[:,0],90):.1f}/{r[:,0].max():.1f}; max stream_end p50 {np.median(r[:,1]):.1f}; med stream_end p50 {np.median(r[:,2]):.1f}; last start max {r[:,9].max():.1f}")
for x in r[np.argsort(r[:,0])][-6:]:
    print("  span %.1f maxSE %.1f medSE %.1f | last CTA %d: SE %.1f wait %.1f->%.1f pub %.1f end %.1f" % tuple(x[:9]))
