"""Is per-CTA speed a property of the SM or of the addresses it streams? c2 static, traced:
(a) 6 launches as is; (b) the same ranges over K/V shifted by `off` bytes in memory."""
import os, sys
import numpy as np, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth, paper_2405_10480_b200 as la
p = synth.config("c2")
q = synth.gen_q(p, "cuda")
k0 = synth.fill_kv_cache(p, "k", "cuda"); v0 = synth.fill_kv_cache(p, "v", "cuda")
plan = la.Plan(1, 32, 32, 128, p.ctx_lens, trace=True)
rows = plan.export()
iters = np.bincount(rows[:, 0], weights=rows[:, 3] - rows[:, 2], minlength=148)
def run(k, v, reps=6):
    sp, sm = [], []
    for r in range(reps + 2):
        torch.cuda.synchronize(); plan.decode(q, k, v); tr = plan.trace().astype(np.int64)
        if r < 2: continue
        dur = (tr[:, 5] - tr[:, 1]) / 1e3
        sp.append(iters * 65536 / dur / 1e3); sm.append(tr[:, 0].copy())
    return np.array(sp), np.array(sm)
A, smA = run(k0, v0)
print("blockIdx->smid stable across launches:", all((smA[i] == smA[0]).all() for i in range(len(smA))))
def corr(X):
    c = np.corrcoef(X); return c[~np.eye(len(X), dtype=bool)].mean()
print("per-CTA speed run-to-run corr: %.2f  spread %.1f..%.1f" % (corr(A), A.mean(0).min(), A.mean(0).max()))
for off_mb in (1, 7, 64):
    off = off_mb * 1024 * 1024 // 2
    kb = torch.empty(k0.numel() + off, dtype=k0.dtype, device="cuda"); kb[off:] = k0.reshape(-1)
    vb = torch.empty(v0.numel() + off, dtype=v0.dtype, device="cuda"); vb[off:] = v0.reshape(-1)
    B, smB = run(kb[off:].view_as(k0), vb[off:].view_as(v0))
    # per-smid comparison
    sa = np.zeros(148); sb = np.zeros(148)
    sa[smA[0]] = A.mean(0); sb[smB[0]] = B.mean(0)
    print(f"shift {off_mb} MB: per-CTA corr base vs shifted %.2f ; per-SMID corr %.2f ; shifted run-to-run %.2f" %
          (np.corrcoef(A.mean(0), B.mean(0))[0, 1], np.corrcoef(sa, sb)[0, 1], corr(B)))
    del kb, vb
