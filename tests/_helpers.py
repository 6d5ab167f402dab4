"""Shared test helpers: run the CUDA path through the C-ABI binding, run the oracle on the
same seeded inputs (regenerated on the host -- never copied from the device), and the
parity gates of DESIGN.md (readings C20, C21)."""
from __future__ import annotations

import math

import numpy as np
import torch

import oracle
import synth

# Gates: BASELINE.json north star tolerance for bf16/fp16 inputs
# with fp32 accumulation, made well-defined per output row (C20), plus the coverage gate
# on L (C21) that a dropped or duplicated LeanTile would fail.
MAX_ABS = 2e-3
MAX_REL = 1e-2
L_ABS = 1e-5


def gate(O_gpu, L_gpu, O_ref, L_ref, max_abs=MAX_ABS, max_rel=MAX_REL, l_abs=L_ABS, what=""):
    O_gpu = np.asarray(O_gpu, dtype=np.float64)
    O_ref = np.asarray(O_ref, dtype=np.float64)
    assert np.all(np.isfinite(O_gpu)), f"{what}: non-finite output"
    err = np.abs(O_gpu - O_ref)
    assert err.max() <= max_abs, f"{what}: max abs err {err.max():.3e}"
    rows_err = err.reshape(-1, O_ref.shape[-1]).max(axis=1)
    rows_mag = np.abs(O_ref).reshape(-1, O_ref.shape[-1]).max(axis=1)
    rel = rows_err / np.maximum(rows_mag, 1e-30)
    assert rel.max() <= max_rel, f"{what}: normwise row rel err {rel.max():.3e}"
    if L_gpu is not None:
        lerr = np.abs(np.asarray(L_gpu, dtype=np.float64) - np.asarray(L_ref, dtype=np.float64))
        assert lerr.max() <= l_abs, f"{what}: max |L err| {lerr.max():.3e}"
    return float(err.max())


def cuda_inputs(p: synth.Problem, device="cuda", token_range=None):
    q = synth.gen_q(p, device)
    k = synth.fill_kv_cache(p, "k", device, token_range=token_range)
    v = synth.fill_kv_cache(p, "v", device, token_range=token_range)
    return q, k, v


def run_cuda(p: synth.Problem, inputs=None, **plan_kw):
    """Decode through the C-ABI (la_plan + la_decode); returns (O, L, plan) on the host."""
    import paper_2405_10480_b200 as la
    q, k, v = inputs if inputs is not None else cuda_inputs(p)
    lens = p.ctx_lens
    if p.q_len > 1:
        plan_kw = dict(plan_kw, q_len=p.q_len)
    if p.layout == "paged":
        bt, num_pages = synth.paged_meta(p)
        plan_kw = dict(plan_kw, block_table=bt, page_size=p.page_size, num_pages=num_pages)
    if p.dtype == "fp8":
        plan_kw = dict(plan_kw, k_scale=p.k_scale, v_scale=p.v_scale)
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, lens, dtype=p.dtype, layout=p.layout,
                   max_ctx=p.max_ctx if p.layout == "bhsd" else 0, **plan_kw)
    out, lse = plan.decode(q, k, v)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), lse.cpu().numpy().astype(np.float64), plan


def kv_f64(p: synth.Problem, x: torch.Tensor, which: str):
    """The cache values the oracle sees: FP8 codes decoded by the oracle's own E4M3 decoder
    (the format definition) times the per-tensor scale (reading C23); else an exact upcast."""
    if p.dtype == "fp8":
        return oracle.dequantize(x.detach().cpu().view(torch.uint8).numpy(), p.k_scale if which == "k" else p.v_scale)
    return synth.to_f64(x)


def run_oracle(p: synth.Problem, causal: bool = True):
    """Full oracle on host-generated inputs (small problems)."""
    q = synth.to_f64(synth.gen_q(p))
    k = kv_f64(p, synth.fill_kv_cache(p, "k"), "k")
    v = kv_f64(p, synth.fill_kv_cache(p, "v"), "v")
    if p.q_len > 1:
        bt = synth.paged_meta(p)[0] if p.layout == "paged" else None
        return oracle.decode_attention_multi(q, k, v, p.ctx_lens, p.scale, causal, p.layout, block_table=bt,
                                             page_size=p.page_size)
    if p.layout == "paged":
        bt, _ = synth.paged_meta(p)
        return oracle.decode_attention(q, k, v, p.ctx_lens, p.scale, "paged", block_table=bt,
                                       page_size=p.page_size)
    return oracle.decode_attention(q, k, v, p.ctx_lens, p.scale, p.layout)


def oracle_unit(p: synth.Problem, b: int, h: int):
    """Oracle output of one work unit (b, h_kv) -- for sampled checks at full size."""
    q = synth.to_f64(synth.gen_q(p))[b, h * p.group:(h + 1) * p.group]
    k = kv_f64(p, synth.gen_kv_unit(p, b, h, "k"), "k")
    v = kv_f64(p, synth.gen_kv_unit(p, b, h, "v"), "v")
    return oracle.decode_attention_unit(q, k, v, p.scale)


def census_expect(p: synth.Problem, b: int):
    """Closed form of the D3 census input: O_c = C #{t : (t // T_c) mod d == c} / n, L = ln n."""
    n = p.ctx_lens[b]
    tc = synth._census_block(p, n)
    C = float(n // tc) if n % tc == 0 else 1.0
    t = np.arange(n)
    counts = np.bincount((t // tc) % p.head_dim, minlength=p.head_dim)
    return C * counts / n, math.log(n)
