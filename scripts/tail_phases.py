"""Where the kernel's tail goes after the last CTA streams its last LeanTile (DESIGN §6 "Epilogue
tail"): per-CTA stream end (trace field t_stream_end), host wait, host fold, end, from one
traced launch after 10 back-to-back ones.

  python scripts/tail_phases.py CFG ENGINE [Q_LEN] [SCHEDULE]     e.g. c3 tcgen05 4
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, synth, paper_2405_10480_b200 as la
cfg, engine = sys.argv[1], sys.argv[2]
qlen = int(sys.argv[3]) if len(sys.argv) > 3 else 1
sched = sys.argv[4] if len(sys.argv) > 4 else "streamk"
p = synth.config(cfg, **(dict(q_len=qlen) if qlen > 1 else {}))
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, trace=True, engine=engine, schedule=sched, q_len=qlen)
for _ in range(10): plan.decode(q, k, v)
torch.cuda.synchronize()
tr = plan.trace().astype(np.int64)
t0 = tr[:, 1].min()
rel = lambda x: np.where(x > 0, (x - t0) / 1e3, np.nan)
st, pub, w0, w1, en, se = rel(tr[:, 1]), rel(tr[:, 2]), rel(tr[:, 3]), rel(tr[:, 4]), rel(tr[:, 5]), rel(tr[:, 6])
print(f"== {cfg} {engine} q{qlen} {sched}: span {np.nanmax(en):.1f}  stream_end min/med/max {np.nanmin(se):.1f}/{np.nanmedian(se):.1f}/{np.nanmax(se):.1f}")
print("   (end - stream_end) med/p90/max %.2f/%.2f/%.2f" % (np.nanmedian(en - se), np.nanpercentile(en - se, 90), np.nanmax(en - se)))
if sched == "streamk":
    hw = w1 - w0
    print("   host wait (w1-w0) med/max %.2f/%.2f ; host fold (pub-w1) med/max %.2f/%.2f ; wait begin - stream_end med %.2f" % (
        np.nanmedian(hw), np.nanmax(hw), np.nanmedian(pub - w1), np.nanmax(pub - w1), np.nanmedian(w0 - se)))
for g in np.argsort(np.nan_to_num(en))[-6:]:
    print(f"   CTA {g:3d}: start {st[g]:.2f} stream_end {se[g]:.1f} publish {pub[g]:.1f} wait {w0[g]:.1f}->{w1[g]:.1f} end {en[g]:.1f}")
