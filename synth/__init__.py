"""Seeded synthetic decode-attention inputs, shared by tests, ``smoke()`` and ``bench.py``.

This module holds NONE of the method's arithmetic (no scores, softmax, rescaling or
scheduling).  It only manufactures Q/K/V values.  Both the CUDA path and the fp64 oracle
consume what it produces; neither imports the other.

Generator
---------
A counter-based generator: every element is a pure function of
``(seed, tensor_id, element coordinates)``, built from a 32-bit multiply/xor-shift hash
evaluated with int64 torch ops whose intermediate products stay below 2**63 (so CPU and
CUDA produce identical bits).  Two hashes per element give four 16-bit uniforms;
their Irwin-Hall sum, centred and scaled by sqrt(3), is an (approximately) standard
normal variate.  All real arithmetic is fp64 with exactly-representable operands
(sums of multiples of 2**-16) followed by one correctly-rounded multiply, then the value
is rounded fp64 -> fp32 -> storage dtype (RNE).  Because every step is either integer or a
single correctly-rounded IEEE operation, a K/V slab generated on the GPU box's device and
the same slab regenerated on the host for the oracle are bit-identical.  That is what
lets the full-size parity tests check sampled outputs without ever copying an input (or an
expected value) from the CUDA path to the oracle.

Distributions
--------------------------------------------------------
* ``D0`` iid:        q, k, v ~ N(0, 1)
* ``D1`` structured: q ~ 2 N(0,1); k ~ N(0,1); v = mu[b,h,c] + 0.5 N(0,1), mu ~ U(-1, 1)
                     (score std ~ 2 -> peaky softmax, |O| ~ 0.5; the default)
* ``D2`` needle:     D1 plus needles: k_t += beta * q_hat at chosen tokens, beta giving a
                     +6 score bump (forces the running max to move across CTAs)
* ``D3`` census:     q = 0; v[t, c] = C * [c == (t // T_c) mod d] (exact closed form output)
* ``D4`` monotone:   D1 with k_t += alpha (t / n) q_hat (running max changes every tile)

Tensor ids: q=0, k=1, v=2, mu=3, needle positions=4.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

_M32 = 0xFFFFFFFF
_DTYPES = {"bf16": torch.bfloat16, "fp16": torch.float16, "fp32": torch.float32, "fp8": torch.float8_e4m3fn}
DTYPE_BYTES = {"bf16": 2, "fp16": 2, "fp32": 4, "fp8": 1}   # K/V bytes per element
Q_DTYPE = {"bf16": "bf16", "fp16": "fp16", "fp32": "fp32", "fp8": "bf16"}  # FP8 KV keeps a bf16 q
E4M3_MAX = 448.0


def _hash32_int(x: int) -> int:
    """Scalar twin of :func:`_hash32` (python ints)."""
    x &= _M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & _M32
    x ^= x >> 15
    x = (x * 0x68E31DA5) & _M32
    x ^= x >> 16
    return x


def _hash32(x: torch.Tensor) -> torch.Tensor:
    """32-bit avalanche hash on an int64 tensor holding values in [0, 2**32)."""
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x68E31DA5) & _M32
    x = x ^ (x >> 16)
    return x


def _key(seed: int, tensor_id: int) -> int:
    return _hash32_int(_hash32_int(seed * 0x9E3779B1) ^ (tensor_id * 0x85EBCA77))


def _normal_from_index(idx: torch.Tensor, key: int) -> torch.Tensor:
    """Approximately N(0,1) fp64 values from int64 element indices (any size)."""
    lo = idx & _M32
    hi = idx >> 32
    h1 = _hash32(lo ^ _hash32(hi ^ key))
    h2 = _hash32(h1 ^ 0x5BD1E995)
    s = ((h1 & 0xFFFF) + (h1 >> 16) + (h2 & 0xFFFF) + (h2 >> 16)).to(torch.float64)
    # four uniforms (u_j = (k_j + 0.5) / 65536) summed: (s + 2) / 65536, mean 2, var 1/3
    return ((s + 2.0) * (1.0 / 65536.0) - 2.0) * math.sqrt(3.0)


def _uniform_from_index(idx: torch.Tensor, key: int) -> torch.Tensor:
    """U[0,1) fp64 values from int64 element indices."""
    lo = idx & _M32
    hi = idx >> 32
    h = _hash32(lo ^ _hash32(hi ^ key))
    return (h.to(torch.float64) + 0.5) * (1.0 / 4294967296.0)


def _round(x64: torch.Tensor, dtype: str) -> torch.Tensor:
    """fp64 -> fp32 -> storage dtype, each a correctly rounded (RNE) cast (E4M3: saturated
    to +-448 first -- torch's cast would turn out-of-range values into NaN)."""
    x32 = x64.to(torch.float32)
    if dtype == "fp8":
        x32 = x32.clamp(-E4M3_MAX, E4M3_MAX)
    return x32.to(_DTYPES[dtype])


@dataclass
class Problem:
    """One decode-attention problem (N_q = 1), the paper's (B, h, N_k, d).

    ``ctx_lens[b]`` is request b's context length.  ``group = heads_q // heads_kv``
    q-heads share KV head ``h_q // group`` (reading C3).
    """

    batch: int
    heads_q: int
    heads_kv: int
    head_dim: int
    ctx_lens: List[int]
    dtype: str = "bf16"
    dist: str = "D1"
    seed: int = 1000
    layout: str = "bhsd"          # "bhsd" (B, H_kv, max_ctx, d) or "packed" (H_kv, sum n, d)
    max_ctx: Optional[int] = None  # bhsd row stride; default max(ctx_lens)
    needles: Sequence[int] = field(default_factory=tuple)  # extra needle tokens (D2)
    census_block: int = 0          # T_c for D3 (0 -> n_b // 16 rounded to a power of two)
    page_size: int = 0             # layout "paged": tokens per page (pools (pages, H_kv, page, d))
    q_len: int = 1                 # N_q query tokens per request (q: (B, H_q, N_q, d) if > 1)
    q_lens: Optional[Sequence[int]] = None  # per-request N_b (heterogeneous batch): q is then
                                            # (sum_b H_q N_b, d), request blocks (H_q, N_b, d)
    k_scale: Optional[float] = None  # dtype "fp8": stored code = value / scale (E4M3, RNE,
    v_scale: Optional[float] = None  # saturating); the cache IS code x scale.  Defaults below.

    def __post_init__(self):
        if self.max_ctx is None:
            self.max_ctx = max(self.ctx_lens)
        # FP8 defaults: amax-style per-tensor scales (non powers of two, so a dropped scale
        # cannot hide); the census's integer V uses 1/2 so its codes stay exact
        if self.k_scale is None:
            self.k_scale = 0.0123 if self.dtype == "fp8" else 1.0
        if self.v_scale is None:
            self.v_scale = (0.5 if self.dist == "D3" else 0.0171) if self.dtype == "fp8" else 1.0
        assert len(self.ctx_lens) == self.batch
        assert self.heads_q % self.heads_kv == 0

    @property
    def group(self) -> int:
        return self.heads_q // self.heads_kv

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.head_dim)

    @property
    def kv_bytes(self) -> int:
        """Algorithmic K+V bytes: 2 * H_kv * sum(n_b) * d * sizeof(kv)."""
        return 2 * self.heads_kv * sum(self.ctx_lens) * self.head_dim * DTYPE_BYTES[self.dtype]

    @property
    def cu_seqlens(self) -> List[int]:
        out = [0]
        for n in self.ctx_lens:
            out.append(out[-1] + n)
        return out


# ----------------------------------------------------------------------------------------
# element generators (all return fp64 tensors before rounding)
# ----------------------------------------------------------------------------------------

def q_row_of(p: Problem, b: int, hq: int, i: int = 0) -> int:
    """Row of query token i of q-head hq of request b in the flat (rows, d) view of q."""
    qls = list(p.q_lens) if p.q_lens is not None else [p.q_len] * p.batch
    return sum(p.heads_q * n for n in qls[:b]) + hq * qls[b] + i


def _q64(p: Problem, device) -> torch.Tensor:
    B, H, D = p.batch, p.heads_q, p.head_dim
    if p.q_lens is not None:
        shape = (H * sum(p.q_lens), D)
    else:
        shape = (B, H, D) if p.q_len == 1 else (B, H, p.q_len, D)
    if p.dist == "D3":
        return torch.zeros(shape, dtype=torch.float64, device=device)
    idx = torch.arange(math.prod(shape), dtype=torch.int64, device=device)
    x = _normal_from_index(idx, _key(p.seed, 0)).reshape(shape)
    if p.dist in ("D1", "D2", "D4"):
        x = x * 2.0
    return x


def gen_q(p: Problem, device="cpu") -> torch.Tensor:
    """Q as (B, H_q, d) in the storage dtype (bf16 for an FP8 KV cache)."""
    return _round(_q64(p, device), Q_DTYPE[p.dtype])


def _qhat_for_unit(p: Problem, b: int, h: int, device) -> torch.Tensor:
    """Unit vector along the (rounded) query of the group's first q-head, fp64."""
    q = gen_q(p, device).reshape(-1, p.head_dim)[q_row_of(p, b, h * p.group)].to(torch.float64)
    # (the first query token of the group's first head)
    nrm = torch.linalg.vector_norm(q)
    return q / nrm, float(nrm)


def _needle_tokens(p: Problem, b: int, h: int) -> List[int]:
    n = p.ctx_lens[b]
    r = _hash32_int(_key(p.seed, 4) ^ (b * 0x27D4EB2F) ^ (h * 0x165667B1)) % n
    toks = {0, n - 1, r}
    toks.update(t for t in p.needles if 0 <= t < n)
    return sorted(toks)


def _census_block(p: Problem, n: int) -> int:
    if p.census_block:
        return p.census_block
    tc = 1
    while tc * 2 <= max(1, n // 16):
        tc *= 2
    return tc


def gen_kv_unit(p: Problem, b: int, h: int, which: str, device="cpu",
                t0: int = 0, t1: Optional[int] = None) -> torch.Tensor:
    """Rows [t0, t1) of K or V for work unit (b, h_kv) as (t1-t0, d) in the storage dtype.

    Element (b, h, t, c) uses index ((b*H_kv + h) << 32) + t*d + c, so a slab is
    layout-independent and can be regenerated piecewise.
    """
    n = p.ctx_lens[b]
    D = p.head_dim
    if t1 is None:
        t1 = n
    assert 0 <= t0 <= t1 <= n
    base = (b * p.heads_kv + h) << 32
    t = torch.arange(t0, t1, dtype=torch.int64, device=device)
    c = torch.arange(D, dtype=torch.int64, device=device)
    idx = base + t[:, None] * D + c[None, :]
    if which == "k":
        x = _normal_from_index(idx, _key(p.seed, 1))
        if p.dist in ("D2", "D4"):
            qhat, qn = _qhat_for_unit(p, b, h, device)
            if p.dist == "D2":
                beta = 6.0 / (p.scale * qn)
                for tok in _needle_tokens(p, b, h):
                    if t0 <= tok < t1:
                        x[tok - t0] += beta * qhat
            else:
                alpha = 8.0 / (p.scale * qn)
                x = x + (alpha * (t.to(torch.float64) / n))[:, None] * qhat[None, :]
        return _round(x / p.k_scale, p.dtype) if p.dtype == "fp8" else _round(x, p.dtype)
    if which == "v":
        if p.dist == "D3":
            tc = _census_block(p, n)
            C = float(n // tc) if n % tc == 0 else 1.0
            hit = ((t // tc) % D)[:, None] == c[None, :]
            return _round(hit.to(torch.float64) * (C / p.v_scale), p.dtype)
        x = _normal_from_index(idx, _key(p.seed, 2))
        if p.dist != "D0":
            mu_idx = ((b * p.heads_kv + h) * D + c)
            mu = _uniform_from_index(mu_idx, _key(p.seed, 3)) * 2.0 - 1.0
            x = mu[None, :] + 0.5 * x
        return _round(x / p.v_scale, p.dtype) if p.dtype == "fp8" else _round(x, p.dtype)
    raise ValueError(which)


def fill_kv_cache(p: Problem, which: str, device="cpu", chunk_rows: int = 1 << 20,
                  token_range=None) -> torch.Tensor:
    """The whole K or V cache in the problem's layout.

    bhsd:   (B, H_kv, max_ctx, d); rows t >= n_b are zero (never read by the method).
    packed: (H_kv, sum_b n_b, d), request b at rows cu_seqlens[b] .. cu_seqlens[b+1].

    ``token_range`` (per request ``(a, b)``) keeps only tokens [a, b) of each request --
    a sequence shard -- laid out as a cache of lengths ``b - a`` (max_ctx = max length).
    """
    D = p.head_dim
    if p.layout == "paged":
        assert token_range is None, "sequence shards of a paged cache are not generated"
        return _fill_paged(p, which, device, chunk_rows)
    if token_range is None:
        token_range = [(0, n) for n in p.ctx_lens]
    lens = [b - a for a, b in token_range]
    max_ctx = p.max_ctx if lens == list(p.ctx_lens) else max(lens)
    if p.layout == "bhsd":
        out = torch.zeros(p.batch, p.heads_kv, max_ctx, D, dtype=_DTYPES[p.dtype], device=device)
    elif p.layout == "packed":
        out = torch.zeros(p.heads_kv, sum(lens), D, dtype=_DTYPES[p.dtype], device=device)
    else:
        raise ValueError(p.layout)
    cu = [0]
    for n in lens:
        cu.append(cu[-1] + n)
    for b in range(p.batch):
        a0, a1 = token_range[b]
        for h in range(p.heads_kv):
            for t0 in range(a0, a1, chunk_rows):
                t1 = min(a1, t0 + chunk_rows)
                slab = gen_kv_unit(p, b, h, which, device, t0, t1)
                r0, r1 = t0 - a0, t1 - a0
                if p.layout == "bhsd":
                    out[b, h, r0:r1] = slab
                else:
                    out[h, cu[b] + r0: cu[b] + r1] = slab
    return out


def paged_meta(p: Problem, spare_pages: int = 3):
    """Block table of a paged problem: the sum_b ceil(n_b / page) used pages plus a few spare
    ones, handed out in a seeded random order (pages of one request are NOT contiguous).
    Returns (block_table int32 [B, pages_per_seq], num_pages)."""
    import numpy as np
    ps = p.page_size
    need = [-(-n // ps) for n in p.ctx_lens]
    num_pages = sum(need) + spare_pages
    order = torch.argsort(_uniform_from_index(torch.arange(num_pages, dtype=torch.int64), _key(p.seed, 5)))
    bt = np.full((p.batch, max(need)), num_pages - 1, dtype=np.int32)   # unused slots: a valid page
    pos = 0
    for b, k in enumerate(need):
        bt[b, :k] = order[pos:pos + k].numpy()
        pos += k
    return bt, num_pages


def _fill_paged(p: Problem, which: str, device, chunk_rows: int):
    bt, num_pages = paged_meta(p)
    ps = p.page_size
    out = torch.zeros(num_pages, p.heads_kv, ps, p.head_dim, dtype=_DTYPES[p.dtype], device=device)
    for b in range(p.batch):
        n = p.ctx_lens[b]
        for h in range(p.heads_kv):
            for t0 in range(0, n, chunk_rows):
                t1 = min(n, t0 + chunk_rows)
                slab = gen_kv_unit(p, b, h, which, device, t0, t1)
                for pi in range(t0 // ps, -(-t1 // ps)):
                    a0, a1 = max(t0, pi * ps), min(t1, (pi + 1) * ps)
                    out[int(bt[b, pi]), h, a0 - pi * ps:a1 - pi * ps] = slab[a0 - t0:a1 - t0]
    return out


def to_f64(x: torch.Tensor):
    """Exact upcast of a storage-dtype tensor to a float64 numpy array."""
    return x.detach().to("cpu").to(torch.float64).numpy()


# ----------------------------------------------------------------------------------------
# the BASELINE.json configurations (SURVEY.md §8(d) "Configs as concrete runs")
# ----------------------------------------------------------------------------------------

C4_CTX_LENS = [131072, 1024, 16586, 17950, 26213, 19032, 99749, 50527, 46403, 81742,
               120314, 109887, 60115, 17344, 107557, 73913]


def config(name: str, dist: str = "D1", **kw) -> Problem:
    """BASELINE.json configs[0..4] as Problems (seed = 1000 + config index); ``dtype=`` may
    override the storage type (e.g. "fp8" for the FP8-KV variant of a workload)."""
    shapes = {
        "c1": ((1, 1, 1, 64, [4096]), "fp32", 1001),
        "c2": ((1, 32, 32, 128, [262144]), "bf16", 1002),
        "c3": ((8, 64, 8, 128, [65536] * 8), "bf16", 1003),
        "c4": ((16, 32, 32, 128, list(C4_CTX_LENS)), "bf16", 1004),
        "c5": ((1, 32, 32, 128, [1 << 20]), "bf16", 1005),
    }
    if name in shapes:
        args, dtype, seed = shapes[name]
        kw.setdefault("dtype", dtype)
        return Problem(*args, dist=dist, seed=seed, **kw)
    raise ValueError(name)


def shard_bounds(p: Problem, rank: int, world: int):
    """Sequence shard ``rank`` of ``world``: request b keeps tokens
    [floor(r n_b / P), floor((r+1) n_b / P)) (contiguous 1/P of every head's context)."""
    return [((rank * n) // world, ((rank + 1) * n) // world) for n in p.ctx_lens]
