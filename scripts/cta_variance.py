"""Per-CTA streaming-time spread of stream-K on c3 (DESIGN §6 "In-flight window"): mean, std,
run-to-run std over 6 traced samples (3 back-to-back launches each), by segment count, slowest /
fastest CTAs with their SM ids.  LEANATTN_LIB selects a library variant.

  python scripts/cta_variance.py
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, synth, paper_2405_10480_b200 as la
p = synth.config("c3")
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
for eng in ("tcgen05", "mma"):
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, trace=True, engine=eng, schedule="streamk")
    seg = plan.export()
    nseg = np.bincount(seg[:, 0], minlength=148)
    first_nonhost = np.zeros(148, bool)
    for g in range(148):
        r = seg[seg[:, 0] == g]
        first_nonhost[g] = r[0, 4] == 0
    S = []
    for rep in range(6):
        for _ in range(3): plan.decode(q, k, v)
        torch.cuda.synchronize()
        tr = plan.trace().astype(np.int64)
        S.append((tr[:, 6] - tr[:, 1]) / 1e3)
    S = np.array(S); s = S.mean(0)
    sm = tr[:, 0]
    print(f"== {eng}: stream time mean {s.mean():.1f} std {s.std():.2f} min {s.min():.1f} max {s.max():.1f}; run-to-run std {S.std(0).mean():.2f}")
    for ns in sorted(set(nseg)):
        m = nseg == ns
        print(f"   segments {ns}: n {m.sum()} mean {s[m].mean():.1f}")
    print(f"   first seg non-host: {s[first_nonhost].mean():.1f} (n {first_nonhost.sum()}), host-first: {s[~first_nonhost].mean():.1f}")
    # position within unit / unit id
    order = np.argsort(s)
    print("   slowest 8 CTAs:", order[-8:], "smid", sm[order[-8:]], np.round(s[order[-8:]], 1))
    print("   fastest 8 CTAs:", order[:8], "smid", sm[order[:8]], np.round(s[order[:8]], 1))
    # smid parity / TPC effect
    for name, m in (("even smid", sm % 2 == 0), ("odd smid", sm % 2 == 1)):
        print(f"   {name}: {s[m].mean():.1f}")
    np.save(f"gpurun_out/cta_variance_{eng}.npy", np.stack([s, sm, nseg]))
