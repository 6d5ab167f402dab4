"""Sequence-sharded multi-GPU decode (BASELINE.json north star, config c5).

Each rank (one process per GPU, ``torch.distributed`` over NCCL/NVLink) holds a contiguous
1/P slice of every head's context, runs the SAME single-GPU kernel on it
(``la_decode_partial`` -> normalised O_r and logsumexp L_r, written into ONE packed buffer),
one all-gather exchanges the per-head (O_r, L_r) pairs (B*H_q*(d+1)*4 bytes per rank: 16.5 KB
at c5), and ``la_combine_strided`` folds them with the softmax re-scaling operator (§4.1; exact for any split by
associativity).  Head- or batch-sharded layouts (the paper's tensor parallelism,
P:511) need no collective at all: every rank simply plans and decodes its own units.

``fused`` path: the exchange moves INTO the decode kernel.  Each rank's
plan is built with ``xchg_world = P``; the ranks swap the CUDA IPC handles of their
exchange buffers once (:func:`connect_exchange`), after which every ``plan.decode`` pushes
the rank's normalised shard partials straight into every peer's HBM over NVLink and folds
the P partials in-kernel -- no NCCL launch, no combine kernel (la.h ``la_plan_xchg_*``).

Host-side glue only; the arithmetic runs in libleanattn.so kernels.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard_bounds(ctx_lens: Sequence[int], rank: int, world: int) -> List[Tuple[int, int]]:
    """Tokens [floor(r n / P), floor((r+1) n / P)) of every request for rank r."""
    return [((rank * n) // world, ((rank + 1) * n) // world) for n in ctx_lens]


def gather_packed(packed, group=None):
    """All-gather every rank's packed (O_r, L_r) buffer (rows * (d + 1) fp32: O then L) in
    ONE collective: returns (P, rows * (d + 1)) in rank order.  NCCL: all_gather_into_tensor
    into a preallocated buffer; other backends (gloo, the CPU tests) via all_gather lists."""
    import torch
    import torch.distributed as dist
    P = dist.get_world_size(group)
    packed = packed.reshape(-1).contiguous()
    if dist.get_backend(group) == "nccl":
        out = torch.empty((P, packed.numel()), dtype=packed.dtype, device=packed.device)
        dist.all_gather_into_tensor(out, packed, group=group)
        return out
    parts = [torch.empty_like(packed) for _ in range(P)]
    dist.all_gather(parts, packed, group=group)
    return torch.stack(parts)


def pack_partials(o_part, lse_part):
    """(O_r, L_r) -> one contiguous rows * (d + 1) buffer (O rows, then the L column)."""
    import torch
    d = o_part.shape[-1]
    return torch.cat([o_part.reshape(-1, d).reshape(-1), lse_part.reshape(-1)])


def gather_partials(o_part, lse_part, group=None):
    """All-gather the per-rank (O_r, L_r) with ONE collective on their packed form: returns
    ([P, rows, d], [P, rows]) in rank order."""
    d = o_part.shape[-1]
    rows = lse_part.numel()
    allp = gather_packed(pack_partials(o_part, lse_part), group)
    return allp[:, :rows * d].reshape(-1, rows, d), allp[:, rows * d:]


def sequence_sharded_decode(plan, q, k_shard, v_shard, group=None, stream=None):
    """One decode step of the sequence-sharded path on this rank; returns the full (O, L)
    (replicated on every rank).  ``plan`` must be built for this rank's shard lengths.  The
    kernel writes O_r and L_r straight into ONE packed buffer, one all-gather exchanges it
    (B*H_q*(d+1)*4 bytes per rank), la_combine_strided folds the P parts in place."""
    import torch
    import torch.distributed as dist
    from .leanattn import la_combine_packed
    rows, d = int(plan.info.q_rows), plan.info.head_dim
    packed = torch.empty(rows * (d + 1), dtype=torch.float32, device=q.device)
    o = packed[:rows * d].view(rows, d)
    l = packed[rows * d:]
    plan.decode_partial(q, k_shard, v_shard, o, l, stream=stream)
    allp = gather_packed(packed, group)
    out, lse = la_combine_packed(allp, dist.get_world_size(group), rows, d, stream=stream)
    return out, lse


def exchange_handles(handle: bytes, group=None) -> List[bytes]:
    """All-gather every rank's 64-byte exchange handle, in rank order (any backend)."""
    import torch.distributed as dist
    out: List[bytes] = [b""] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return out


def connect_exchange(plan, group=None) -> None:
    """Open every peer rank's exchange buffer in ``plan`` (built with xchg_world = P and
    xchg_rank = this rank).  Collective: every rank must call it.  If any rank fails to map
    a peer, EVERY rank raises the same RuntimeError (so all ranks can agree on a fallback)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    handles = exchange_handles(plan.xchg_handle(), group)
    err = ""
    for peer, h in enumerate(handles):
        if peer != rank and not err:
            try:
                plan.xchg_open(peer, h)
            except Exception as e:  # noqa: BLE001 -- reported collectively below
                err = f"rank {rank} -> peer {peer}: {e}"
    errs: List[str] = [""] * dist.get_world_size(group)
    dist.all_gather_object(errs, err, group=group)
    bad = [e for e in errs if e]
    if bad:
        raise RuntimeError("exchange setup failed: " + "; ".join(bad))


def fused_sequence_sharded_decode(plan, q, k_shard, v_shard, stream=None):
    """One decode step of the fused path: ``plan`` (this rank's shard, exchange connected)
    returns the full (O, L) on every rank from ONE kernel launch."""
    return plan.decode(q, k_shard, v_shard, stream=stream)
