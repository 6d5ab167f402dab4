"""LeanTile-size sweep on small/medium decode shapes (the auto tile rule's regime):
kernel time with a 512 MB L2 flush before every launch.

  python scripts/sweep_tile.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2405_10480_b200 as la  # noqa: E402

SHAPES = [  # (batch, heads_q, heads_kv, d, ctx, dtype)
    (1, 1, 1, 64, 4096, "fp32"),     # c1, 2 MB
    (1, 8, 8, 128, 2048, "bf16"),    # 8 MB
    (1, 4, 4, 128, 4096, "bf16"),    # 8 MB
    (1, 1, 1, 128, 16384, "bf16"),   # 8 MB
    (4, 8, 8, 128, 1024, "bf16"),    # 16 MB
    (1, 32, 8, 128, 4096, "bf16"),   # GQA 16 MB
    (1, 32, 32, 128, 1024, "bf16"),  # 16 MB
]


def main():
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for (B, Hq, Hk, d, n, dt) in SHAPES:
        p = synth.Problem(B, Hq, Hk, d, [n] * B, dtype=dt)
        q = synth.gen_q(p, "cuda")
        k = synth.fill_kv_cache(p, "k", "cuda")
        v = synth.fill_kv_cache(p, "v", "cuda")
        res = []
        for tn in (0, 32, 64, 128, 256):
            plan = la.Plan(B, Hq, Hk, d, p.ctx_lens, dtype=dt, tile_n=tn)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for r in range(60):
                flush.zero_()
                e0.record()
                plan.decode(q, k, v)
                e1.record()
                torch.cuda.synchronize()
                if r >= 10:
                    ts.append(e0.elapsed_time(e1) * 1e3)
            res.append(f"T{plan.info.tile_n}/G{plan.info.grid}{'*' if tn == 0 else ''} {np.median(ts):.1f}")
            plan.close()
        print(f"B{B} Hq{Hq} Hkv{Hk} d{d} n{n} {dt} {p.kv_bytes / 2**20:.0f} MB: " + "  ".join(res), flush=True)


if __name__ == "__main__":
    main()
