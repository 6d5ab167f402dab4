"""Per-CTA stage accounting from an LA_PROF build (trace fields reused, see decode.cu):
consumer warp 0's cycles waiting for data / inside stage() / stage count, and the producer's
cycles waiting for free ring slots.

  LEANATTN_LIB=.../libleanattn_prof.so python scripts/prof_stages.py c3 tcgen05
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402


def main(cfg, engine, q_len=1):
    p = synth.config(cfg, **(dict(q_len=q_len) if q_len > 1 else {}))
    q = synth.gen_q(p, "cuda")
    k = synth.fill_kv_cache(p, "k", "cuda")
    v = synth.fill_kv_cache(p, "v", "cuda")
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, dtype=p.dtype, layout=p.layout,
                   trace=True, engine=engine, q_len=q_len)
    for _ in range(5):
        plan.decode(q, k, v)
    import torch
    torch.cuda.synchronize()
    tr = plan.trace().astype(np.int64)
    span = (tr[:, 5] - tr[:, 1]) / 1e3
    pw, wait, work, n = tr[:, 0], tr[:, 2], tr[:, 3], tr[:, 4]
    print(f"{cfg} {engine}: CTA span us median {np.median(span):.1f}  stages/warp0 {np.median(n):.0f}")
    print(f"  consumer warp0: wait-for-data cycles/stage {np.median(wait / n):.0f}  in-stage cycles/stage {np.median(work / n):.0f}")
    print(f"  producer: wait-for-slot cycles total median {np.median(pw):.0f} (per stage {np.median(pw) / (np.median(n) * plan.info.stage_tokens and 1):.0f})")
    cyc_span = span * 1.965e3
    loop = (wait + work) / 1.965e3
    print(f"  span us min/median/max {span.min():.1f}/{np.median(span):.1f}/{span.max():.1f};"
          f" stage-loop us min/median/max {loop.min():.1f}/{np.median(loop):.1f}/{loop.max():.1f}")
    o = np.argsort(span)[-6:]
    for g in o:
        print(f"   slow CTA {g}: span {span[g]:.1f} loop {loop[g]:.1f} wait/stage {wait[g] / n[g]:.0f} work/stage {work[g] / n[g]:.0f} n {n[g]}")
    print(f"  warp0 busy fraction {np.median(work / cyc_span):.2f}, waiting fraction {np.median(wait / cyc_span):.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "mma", int(sys.argv[3]) if len(sys.argv) > 3 else 1)
