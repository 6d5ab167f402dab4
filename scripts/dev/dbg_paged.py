import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, synth, oracle
import paper_2405_10480_b200 as la
from test_gpu_update import _oracle_paged_prefix
cap = synth.Problem(3, 4, 4, 128, [4096]*3, dtype="bf16", dist="D1", seed=41, layout="paged", page_size=64)
q = synth.gen_q(cap, "cuda"); k = synth.fill_kv_cache(cap, "k", "cuda"); v = synth.fill_kv_cache(cap, "v", "cuda")
bt, npg = synth.paged_meta(cap)
for lens in ([4096]*3, [3000, 1, 2047], [3000, 2000, 2047]):
    O1, L1 = _oracle_paged_prefix(cap, lens)
    for kw in (dict(), dict(grid=7), dict(tile_n=64)):
        plan = la.Plan(3, 4, 4, 128, lens, layout="paged", block_table=bt, page_size=64, num_pages=npg, **kw)
        o, l = plan.decode(q, k, v); torch.cuda.synchronize()
        print(lens, kw, plan.info.grid, plan.info.num_vctas, "Lerr", np.abs(l.cpu().numpy() - L1).max())
        plan.update(lens); o, l = plan.decode(q, k, v); torch.cuda.synchronize()
        print("  after update Lerr", np.abs(l.cpu().numpy() - L1).max())
