"""GPU: la_decode_partial on sequence shards + la_combine == unsharded attention (oracle).

Single-GPU simulated sharding: the P shards of the sequence-sharded
multi-GPU path are decoded one after another on one device and folded by la_combine."""
import numpy as np
import pytest
import torch

import oracle
import synth
from _helpers import cuda_inputs, gate, oracle_unit, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2405_10480_b200 import build as b
    b.build()


def _sharded(p, P, **plan_kw):
    import paper_2405_10480_b200 as la
    q = synth.gen_q(p, "cuda")
    o_parts, l_parts = [], []
    for r in range(P):
        bounds = synth.shard_bounds(p, r, P)
        lens = [b - a for a, b in bounds]
        k = synth.fill_kv_cache(p, "k", "cuda", token_range=bounds)
        v = synth.fill_kv_cache(p, "v", "cuda", token_range=bounds)
        plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, lens, dtype=p.dtype, **plan_kw)
        o, l = plan.decode_partial(q, k, v)
        o_parts.append(o)
        l_parts.append(l)
        del k, v
    O, L = la.la_combine(torch.stack(o_parts).contiguous(), torch.stack(l_parts).contiguous())
    torch.cuda.synchronize()
    return O.cpu().numpy(), L.cpu().numpy(), [o.cpu().numpy() for o in o_parts], [l.cpu().numpy() for l in l_parts]


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_sharded_equals_oracle(P):
    p = synth.Problem(2, 4, 4, 128, [3000, 1777], dtype="bf16", dist="D2", seed=21)
    O_ref, L_ref = run_oracle(p)
    O, L, o_parts, l_parts = _sharded(p, P)
    gate(O, L, O_ref, L_ref, what=f"sharded P={P}")
    # la_combine alone vs the oracle's combine on the same (fp32) partials
    O2, L2 = oracle.combine_shards(np.stack(o_parts).reshape(P, -1, 128), np.stack(l_parts).reshape(P, -1))
    assert np.max(np.abs(O.reshape(-1, 128) - O2)) <= 1e-5 and np.max(np.abs(L.reshape(-1) - L2)) <= 1e-5


def test_c5_sharded_full_size_sampled():
    """BASELINE.json config 5 (n = 1M) as the 8 shards of an 8-GPU run, on one device."""
    p = synth.config("c5")
    O, L, _, _ = _sharded(p, 8)
    O_ref, L_ref = oracle_unit(p, 0, 5)
    gate(O[0, 5:6], L[0, 5:6], O_ref, L_ref, what="c5 head 5")
    torch.cuda.empty_cache()
