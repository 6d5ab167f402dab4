import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import synth, paper_2405_10480_b200 as la
for cfg in ("c3", "c2"):
    p = synth.config(cfg)
    q = synth.gen_q(p, "cuda"); k = synth.fill_kv_cache(p, "k", "cuda"); v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, trace=True, schedule="dynamic")
    for _ in range(3): plan.decode(q, k, v)
    torch.cuda.synchronize(); plan.decode(q, k, v); tr = plan.trace().astype(np.int64)
    t0 = tr[:, 1].min(); end = (tr[:, 5] - t0) / 1e3
    epi = (tr[:, 0] >> 16) / 1e3
    o = np.argsort(end)[::-1]
    fold = tr[:, 2] * 1.0; nf = tr[:, 2] * 0
    print(cfg, "segments of slowest", [(round(fold[g], 1), int(nf[g])) for g in o[:8]], "segments med", np.median(fold), "epi busy med", np.median((tr[:, 0] >> 16) / 1e3))
    print(cfg, "end med", np.median(end), "max", end.max(), "epi med", np.median(epi), "epilogue busy (us) of slowest", [(round(end[g],1), round(epi[g],1), int(tr[g,3]), int(tr[g,4])) for g in o[:8]])
