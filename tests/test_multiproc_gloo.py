"""N > 1 host logic on CPU: world_size-2 (and 3) `gloo` process groups exercise the
sequence-sharded path's glue (shard bounds, per-rank partial exchange in rank order) with
the oracle standing in for the per-rank GPU kernel; the gathered partials folded by the
oracle's combine must equal unsharded attention."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2405_10480_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.Problem(2, 4, 4, 32, [777, 1500], dtype="bf16", dist="D2", seed=41)
    bounds = sharded.shard_bounds(p.ctx_lens, rank, world)
    assert bounds == synth.shard_bounds(p, rank, world)
    q = synth.to_f64(synth.gen_q(p))
    o_r = np.zeros((p.batch, p.heads_q, p.head_dim))
    l_r = np.zeros((p.batch, p.heads_q))
    for b, (a0, a1) in enumerate(bounds):
        for h in range(p.heads_kv):
            k = synth.to_f64(synth.gen_kv_unit(p, b, h, "k", "cpu", a0, a1))
            v = synth.to_f64(synth.gen_kv_unit(p, b, h, "v", "cpu", a0, a1))
            o, l = oracle.decode_attention_unit(q[b, h:h + 1], k, v, p.scale)
            o_r[b, h], l_r[b, h] = o[0], l[0]
    o_all, l_all = sharded.gather_partials(torch.from_numpy(o_r).float(), torch.from_numpy(l_r).float())
    assert o_all.shape == (world, p.batch * p.heads_q, p.head_dim)
    O, L = oracle.combine_shards(o_all.double().numpy(), l_all.double().numpy())
    if rank == 0:
        O_ref, L_ref = oracle.decode_attention(q, synth.to_f64(synth.fill_kv_cache(p, "k")),
                                               synth.to_f64(synth.fill_kv_cache(p, "v")), p.ctx_lens, p.scale)
        err = max(np.abs(O - O_ref.reshape(-1, p.head_dim)).max(), np.abs(L - L_ref.reshape(-1)).max())
        with open(result_path, "w") as f:
            f.write(repr(float(err)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sequence_sharded_glue_gloo(world, tmp_path):
    result = str(tmp_path / "err.txt")
    mp.spawn(_worker, args=(world, _free_port(), result), nprocs=world, join=True)
    err = float(open(result).read())
    # fp32 exchange of the partials (as on the GPU path) bounds the error
    assert err <= 1e-6


class _FakeXchgPlan:
    """Stands in for a Plan built with xchg_world = P: records which peer handles it opens."""

    def __init__(self, rank):
        self.rank = rank
        self.opened = {}

    def xchg_handle(self):
        return bytes([self.rank]) * 64

    def xchg_open(self, peer, handle):
        self.opened[peer] = handle


def _xchg_worker(rank, world, port, result_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2405_10480_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = _FakeXchgPlan(rank)
    sharded.connect_exchange(plan)
    ok = sorted(plan.opened) == [r for r in range(world) if r != rank] and \
        all(h == bytes([r]) * 64 for r, h in plan.opened.items())
    with open(f"{result_path}.{rank}", "w") as f:
        f.write("ok" if ok else repr(plan.opened))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_exchange_handle_swap_gloo(world, tmp_path):
    """NEXT-2 host glue: every rank opens every OTHER rank's exchange handle, in rank order."""
    result = str(tmp_path / "xchg")
    mp.spawn(_xchg_worker, args=(world, _free_port(), result), nprocs=world, join=True)
    for r in range(world):
        assert open(f"{result}.{r}").read() == "ok"
