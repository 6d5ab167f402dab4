"""GPU parity of the FP8 KV cache (NEXT-4: E4M3 codes + per-tensor scales, bf16 q) through
the C ABI against the fp64 oracle on the dequantised cache (oracle.dequantize: the oracle's
own E4M3 decoder, reading C23).  One tensor-core engine serves every T_m <= 8, so MHA
(g = 1), GQA, N_q > 1, paged and packed layouts all run the same FP8 kernel."""
import numpy as np
import pytest
import torch

import synth
from _helpers import census_expect, cuda_inputs, gate, oracle_unit, run_cuda, run_oracle

pytestmark = pytest.mark.gpu

SCHEDULES = ("streamk", "dynamic")


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_2405_10480_b200 import build as b
    b.build()
    import paper_2405_10480_b200 as la
    la.lib()


@pytest.mark.parametrize("group", [1, 2, 8])
@pytest.mark.parametrize("dist", ["D0", "D1", "D2", "D4"])
def test_fp8_small_multi_tile_ragged(group, dist):
    p = synth.Problem(2, 2 * group, 2, 128, [1000, 777], dtype="fp8", dist=dist, seed=71, max_ctx=1024)
    O_ref, L_ref = run_oracle(p)
    inputs = cuda_inputs(p)
    for schedule in SCHEDULES:
        for tile_n in (32, 128, 256):
            for grid in (1, 3, 0):
                O, L, plan = run_cuda(p, inputs=inputs, tile_n=tile_n, grid=grid, schedule=schedule)
                gate(O, L, O_ref, L_ref, what=f"fp8 g{group}/{dist}/T{tile_n}/G{grid}/{schedule}")


def test_fp8_scales_are_applied():
    # the same codes under other scales: K's scale moves the softmax, V's scales O linearly
    p = synth.Problem(1, 4, 4, 128, [3000], dtype="fp8", dist="D1", seed=72)
    inputs = cuda_inputs(p)
    for ks, vs in ((p.k_scale, p.v_scale), (0.05, 1.0), (0.002, 3.5)):
        p2 = synth.Problem(1, 4, 4, 128, [3000], dtype="fp8", dist="D1", seed=72, k_scale=ks, v_scale=vs)
        O, L, _ = run_cuda(p2, inputs=inputs, grid=0)
        q = synth.to_f64(synth.gen_q(p2))
        import oracle
        codes_k = inputs[1].cpu().view(torch.uint8).numpy()
        codes_v = inputs[2].cpu().view(torch.uint8).numpy()
        O_ref, L_ref = oracle.decode_attention(q, oracle.dequantize(codes_k, ks), oracle.dequantize(codes_v, vs),
                                               p2.ctx_lens, p2.scale)
        gate(O / max(vs, 1.0), L, O_ref / max(vs, 1.0), L_ref, what=f"scales {ks} {vs}")


def test_fp8_census_and_determinism():
    p = synth.Problem(3, 2, 2, 128, [4096, 2048, 1024], dtype="fp8", dist="D3", seed=73, max_ctx=4096)
    O, L, _ = run_cuda(p, tile_n=64, grid=0)
    for b in range(3):
        o_exp, l_exp = census_expect(p, b)
        assert np.max(np.abs(O[b] - o_exp[None, :])) <= 1e-5
        assert np.max(np.abs(L[b] - l_exp)) <= 1e-5
    import paper_2405_10480_b200 as la
    p = synth.Problem(1, 8, 1, 128, [5000], dtype="fp8", dist="D2", seed=74)
    q, k, v = cuda_inputs(p)
    for schedule in SCHEDULES:
        plan = la.Plan(1, 8, 1, 128, [5000], dtype="fp8", grid=11, tile_n=64, schedule=schedule,
                       k_scale=p.k_scale, v_scale=p.v_scale)
        ref = plan.decode(q, k, v)[0].clone()
        for _ in range(5):
            assert torch.equal(plan.decode(q, k, v)[0], ref)


@pytest.mark.parametrize("group", [1, 8])
@pytest.mark.parametrize("page_size", [16, 64, 256])
def test_fp8_paged(group, page_size):
    p = synth.Problem(3, 2 * group, 2, 128, [1000, 77, 2500], dtype="fp8", dist="D2", seed=75,
                      layout="paged", page_size=page_size)
    O_ref, L_ref = run_oracle(p)
    inputs = cuda_inputs(p)
    for schedule in SCHEDULES:
        for tile_n, grid in ((32, 5), (256, 0)):
            O, L, _ = run_cuda(p, inputs=inputs, tile_n=tile_n, grid=grid, schedule=schedule)
            gate(O, L, O_ref, L_ref, what=f"fp8 paged g{group} ps{page_size} T{tile_n} G{grid} {schedule}")


def test_fp8_packed_and_multi_token():
    p = synth.Problem(4, 8, 2, 128, [300, 1500, 64, 999], dtype="fp8", dist="D1", seed=76, layout="packed")
    O_ref, L_ref = run_oracle(p)
    for grid in (3, 0):
        O, L, _ = run_cuda(p, tile_n=64, grid=grid)
        gate(O, L, O_ref, L_ref, what=f"fp8 packed G{grid}")
    for causal in (True, False):
        p = synth.Problem(2, 4, 2, 128, [900, 333], dtype="fp8", dist="D2", seed=77, q_len=2)
        O_ref, L_ref = run_oracle(p, causal=causal)
        O, L, _ = run_cuda(p, tile_n=64, grid=7, causal=causal)
        gate(O, L, O_ref, L_ref, what=f"fp8 Nq2 causal={causal}")


def test_fp8_c2_c3_full_size_sampled():
    """The c2 (MHA 256k) and c3 (GQA 8 x 64k) workloads with an FP8 cache, bench launch config."""
    p = synth.config("c2", dtype="fp8")
    inputs = cuda_inputs(p)
    O, L, plan = run_cuda(p, inputs=inputs)
    assert plan.info.grid == 148 and plan.info.tile_n == 256
    for h in (0, 19):
        O_ref, L_ref = oracle_unit(p, 0, h)
        gate(O[0, h:h + 1], L[0, h:h + 1], O_ref, L_ref, what=f"fp8 c2 head {h}")
    del inputs
    torch.cuda.empty_cache()
    p = synth.config("c3", dtype="fp8")
    O, L, plan = run_cuda(p)
    for b, h in ((0, 0), (5, 3)):
        O_ref, L_ref = oracle_unit(p, b, h)
        gate(O[b, 8 * h:8 * h + 8], L[b, 8 * h:8 * h + 8], O_ref, L_ref, what=f"fp8 c3 b{b} h{h}")
    torch.cuda.empty_cache()
