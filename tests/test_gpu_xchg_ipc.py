"""NEXT-2 exchange set-up across PROCESSES (the default route of `bench.py --gpus N`):
two processes on one GPU swap their exchange buffers' CUDA IPC handles over a gloo group
(la_plan_xchg_handle -> la_plan_xchg_open via sharded.connect_exchange), each then reads
the peer's shape header THROUGH the mapping (la_plan_xchg_open checks it), a plan of another
shape is rejected collectively, and a rank whose peer never launches gets LA_ERR_TIMEOUT
from la_plan_status instead of a hung device."""
import os
import socket

import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_path):
    import faulthandler
    import sys
    import time
    faulthandler.enable()
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import synth
    import paper_2405_10480_b200 as la
    from paper_2405_10480_b200 import sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    log = []

    def note(x):
        log.append(x)
        with open(f"{result_path}.{rank}", "w") as f:
            f.write(" ".join(log))
    p = synth.Problem(1, 4, 4, 128, [4000], dtype="bf16", dist="D1", seed=61)
    bounds = synth.shard_bounds(p, rank, world)
    lens = [b - a for a, b in bounds]
    plan = la.Plan(1, 4, 4, 128, lens, xchg_world=world, xchg_rank=rank, grid=8)
    sharded.connect_exchange(plan)          # opens the peer's buffer and checks its header
    note("open-ok")
    # a plan of another shape on rank 1: every rank must see the set-up fail
    other = la.Plan(1, 4, 4, 128, lens, xchg_world=world, xchg_rank=rank, grid=8) if rank == 0 else \
        la.Plan(1, 8, 8, 128, lens, xchg_world=world, xchg_rank=rank, grid=8)
    try:
        sharded.connect_exchange(other)
        note("mismatch-accepted")
    except RuntimeError as e:
        note("mismatch-rejected" if "header mismatch" in str(e) else f"mismatch-other:{e}")
    dist.barrier()
    if rank == 0:   # the peer never launches: the exchange wait must give up and say so
        q = synth.gen_q(p, "cuda")
        k = synth.fill_kv_cache(p, "k", "cuda", token_range=bounds)
        v = synth.fill_kv_cache(p, "v", "cuda", token_range=bounds)
        t0 = time.time()
        plan.decode(q, k, v)
        try:
            plan.status()
            note("no-timeout")
        except la.LaError as e:
            note("timeout" if e.status == la.LA_ERR_TIMEOUT else f"status-{e.status}")
        note(f"waited {time.time() - t0:.1f}s")
        plan.status()                      # the error word is cleared once reported
        note("cleared")
    dist.barrier()
    note("done")
    dist.destroy_process_group()


def test_ipc_exchange_open_header_check_and_timeout(tmp_path):
    import torch
    assert torch.cuda.is_available()
    result = str(tmp_path / "ipc")
    try:
        mp.spawn(_worker, args=(2, _free_port(), result), nprocs=2, join=True)
    finally:
        for r in range(2):
            if os.path.exists(f"{result}.{r}"):
                print(f"rank {r}:", open(f"{result}.{r}").read())
    r0 = open(f"{result}.0").read().split()
    r1 = open(f"{result}.1").read().split()
    assert r0[:2] == ["open-ok", "mismatch-rejected"] and r1 == ["open-ok", "mismatch-rejected", "done"], (r0, r1)
    assert r0[2] == "timeout" and r0[-2:] == ["cleared", "done"], r0
