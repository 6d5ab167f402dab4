#!/usr/bin/env python
"""bench.py -- LeanAttention decode on B200: latency and achieved HBM GB/s (BASELINE.json).

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config c1..c5]

* N = 1 (default): BASELINE.json configs[1] (c2: batch 1, 32 heads, d 128, context 256k,
  bf16 KV) on one B200 -- the north-star workload.  One step = one la_decode (the whole hot
  path: stream-K LeanTiles + in-kernel fixup + finalize, one launch).
* N > 1 (torchrun, one rank per GPU): configs[4] (c5: context 1M) sequence-sharded --
  every rank decodes its contiguous 1/N of every head's context (la_decode_partial), NCCL
  all-gathers the per-head (O_r, L_r) and la_combine folds them.  Total work is fixed:
  "scaling": "strong".
* --impl reference: the fp64 CPU oracle (oracle/), timed on this host's cores on a bounded
  sample of the same workload (this tier has no runnable reference implementation).

``value`` = algorithmic KV bytes (2 * H_kv * sum n * d * 2 B) / device time, GB/s, whole job.
Inputs (4.3 GB at c2) are larger than the 126 MB L2, so no flush is needed between steps;
configs whose KV fits in L2 are flushed (a 512 MB memset) before every step.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "decode-attention latency (µs) and achieved HBM GB/s vs peak at 1/2/4/8 B200"
WORKLOADS = {
    "c1": "batch 1, 1 head, head_dim 64, context 4096, fp32 inputs",
    "c2": "batch 1, 32 heads, head_dim 128, context 256k, bf16 KV cache, 1 B200",
    "c3": "batch 8, 64 q-heads / 8 kv-heads (GQA), head_dim 128, context 64k, bf16",
    "c4": "batch 16, 32 heads, head_dim 128, ragged context lengths 1k-128k per request",
    "c5": "batch 1, 32 heads, head_dim 128, context 1M, KV sequence-sharded across N B200 (partials exchanged and combined across GPUs)",
}
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=None, help="c1..c5 (default c2 at N=1, c5 at N>1)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-heads", type=int, default=32, help="heads in the oracle cpu_baseline sample")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--schedule", default="auto", choices=["auto", "streamk", "dynamic", "sequential", "fixed_split"])
    ap.add_argument("--page-size", type=int, default=0, help="run the config in a paged KV pool (16..256)")
    ap.add_argument("--engine", default="auto", choices=["auto", "mma", "tcgen05"],
                    help="tensor-core engine for T_m > 1 tiles (GQA): auto (the plan's rule), mma.sync or tcgen05 + TMEM")
    ap.add_argument("--q-len", type=int, default=1,
                    help="N_q query tokens per request (speculative decode; single GPU, no e2e / cpu legs)")
    ap.add_argument("--tile-n", type=int, default=0, help="LeanTile size T_n (0 = planner's auto rule)")
    ap.add_argument("--dtype", default=None, choices=["bf16", "fp16", "fp8"],
                    help="KV storage type (default: the config's; fp8 = E4M3 codes + scales, bf16 q; NEXT-4)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo only to test the multi-rank path on one GPU)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "p2p"],
                    help="N > 1: the fused in-kernel NVLink exchange (p2p, NEXT-2) or NCCL all-gather + "
                         "la_combine; auto = p2p on the nccl backend")
    ap.add_argument("--sm-weights", default="off", choices=["off", "calibrate"],
                    help="stream-K plans: SM-rate-weighted ranges from la_plan_calibrate (before the warm-up)")
    ap.add_argument("--dyn-first", type=int, default=940, help="dynamic schedule: head share of each range (permille)")
    ap.add_argument("--dyn-min", type=int, default=2, help="dynamic schedule: smallest virtual CTA (LeanTiles)")
    return ap.parse_args()


# --------------------------------------------------------------------------------------
# clocks during the timed region (NVML)
# --------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            self._nv = None
            self.error = str(e)

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h) \
                    if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self._nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": getattr(self, "error", "")}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


# --------------------------------------------------------------------------------------
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy, read+write bytes)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_probe_gbs():
    """Measured pure streaming-read ceiling (scripts/read_probe.cu, profiles/read_probe.json):
    context for the roofline, not the contract's denominator."""
    path = os.path.join(ROOT, "profiles", "read_probe.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    return max(r["GBps"] for r in d["results"] if r["probe"] == "tma_bulk_ring")


def ncu_traffic(config: str):
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    ent = d.get(config)
    return None if ent is None else ent.get("dram_bytes_per_launch")


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        return 1


def oracle_sample(p, heads, tokens=None, device="cuda"):
    """Host fp64 inputs for the oracle's bounded sample: the first `heads` units, optionally
    only their first `tokens` keys.  Generated by synth (bit-identical on any device)."""
    import synth
    units = []
    q_all = synth.gen_q(p, "cpu")
    for u in range(heads):
        b, h = divmod(u, p.heads_kv)
        n = p.ctx_lens[b] if tokens is None else min(tokens, p.ctx_lens[b])
        k = synth.gen_kv_unit(p, b, h, "k", device, 0, n).cpu()
        v = synth.gen_kv_unit(p, b, h, "v", device, 0, n).cpu()
        units.append((q_all[b, h * p.group:(h + 1) * p.group], k, v))
    return units


def run_oracle_sample(units, scale):
    """The oracle as it stands on the sample (bf16 -> fp64 upcast included)."""
    import numpy as np
    import torch
    import oracle
    t0 = time.perf_counter()
    for q, k, v in units:
        oracle.decode_attention_unit(q.to(torch.float64).numpy(), k.to(torch.float64).numpy(),
                                     v.to(torch.float64).numpy(), scale)
    return time.perf_counter() - t0


def sample_bytes(units, elem=2):
    return sum(2 * k.numel() * elem for _, k, _ in units)


# --------------------------------------------------------------------------------------
def bench_reference(args):
    """--impl reference: the oracle on this host's cores, same metric/unit/config."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import synth
    cfg = args.config or ("c2" if args.gpus == 1 else "c5")
    p = synth.config(cfg)
    dev = "cuda" if _has_cuda() else "cpu"
    # size the per-step sample so that (K + W) steps stay within ~120 s
    probe = oracle_sample(p, 1, tokens=min(p.ctx_lens[0], 1 << 16), device=dev)
    t_probe = run_oracle_sample(probe, p.scale)
    per_token = t_probe / probe[0][1].shape[0]
    budget = 120.0 / max(1, args.steps + args.warmup)
    tokens = int(max(1024, min(p.ctx_lens[0], budget / max(per_token, 1e-12))))
    units = oracle_sample(p, 1, tokens=tokens, device=dev)
    for _ in range(args.warmup):
        run_oracle_sample(units, p.scale)
    t = 0.0
    for _ in range(args.steps):
        t += run_oracle_sample(units, p.scale)
    step_s = t / args.steps
    gbs = sample_bytes(units) / step_s / 1e9
    sample = f"1 of {p.batch * p.heads_kv} (b, h_kv) units of {cfg}, first {tokens} of {p.ctx_lens[0]} tokens"
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3,
            "higher_is_better": True, "scaling": "weak" if args.gpus == 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter-based generator, D1)",
            "config": {"workload": f"{cfg}: {WORKLOADS[cfg]}", "sample": sample},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": blas_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


# --------------------------------------------------------------------------------------
def _timed_loop(step, steps, stream, sync, per_launch=True):
    """K steps between two events.  per_launch: also a (ev0, ev1) pair around each step's
    decode launch (sorted per-launch ms returned; the event records between launches add
    ~5 us per step, so the reported timed region runs without them unless the step holds
    other work, e.g. an L2 flush).  Returns (total_ms / K, sorted per-launch ms or None)."""
    import torch
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)] if per_launch else [None] * steps
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)] if per_launch else [None] * steps
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sync()
    t0.record(stream)
    for i in range(steps):
        step(ev0[i], ev1[i])
    t1.record(stream)
    sync()
    return (t0.elapsed_time(t1) / steps,
            sorted(a.elapsed_time(b) for a, b in zip(ev0, ev1)) if per_launch else None)


def bench_ours(args):
    import torch
    import torch.distributed as dist
    import synth
    import paper_2405_10480_b200 as la
    from paper_2405_10480_b200.leanattn import SCHEDULE_NAMES, la_combine_packed

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    local = local % torch.cuda.device_count()   # --backend gloo tests N ranks on fewer GPUs
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)
    from paper_2405_10480_b200 import sharded

    cfg = args.config or ("c2" if world == 1 else "c5")
    dkw = {"dtype": args.dtype} if args.dtype else {}
    if args.q_len > 1:
        if world > 1:
            raise SystemExit("--q-len is a single-GPU option")
        dkw["q_len"] = args.q_len
        args.no_cpu = args.no_e2e = True
    p = synth.config(cfg, **dkw)
    paged_kw = {}
    if p.dtype == "fp8":
        paged_kw = dict(k_scale=p.k_scale, v_scale=p.v_scale)
    if args.page_size:  # the same workload in a paged pool (NEXT-4); single GPU only
        if world > 1:
            raise SystemExit("--page-size is a single-GPU option")
        p = synth.config(cfg, layout="paged", page_size=args.page_size, **dkw)
        bt, num_pages = synth.paged_meta(p)
        paged_kw.update(block_table=bt, page_size=args.page_size, num_pages=num_pages)
    bounds = synth.shard_bounds(p, rank, world)
    lens = [b - a for a, b in bounds]
    fused = world > 1 and (args.exchange == "p2p" or (args.exchange == "auto" and args.backend == "nccl"))

    q = synth.gen_q(p, dev)
    k = synth.fill_kv_cache(p, "k", dev, token_range=None if args.page_size else bounds)
    v = synth.fill_kv_cache(p, "v", dev, token_range=None if args.page_size else bounds)
    plan_kw = dict(dtype=p.dtype, layout=p.layout, schedule=args.schedule, dyn_first_permille=args.dyn_first,
                   dyn_min_chunk=args.dyn_min, tile_n=args.tile_n, engine=args.engine, q_len=args.q_len, **paged_kw)
    plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, lens, **plan_kw,
                   **(dict(xchg_world=world, xchg_rank=rank) if fused else {}))
    xchg_note = None
    if fused:   # collective decision: every rank maps every peer's buffer, or all use NCCL
        try:
            sharded.connect_exchange(plan)
        except RuntimeError as e:   # raised identically on every rank
            fused = False
            xchg_note = {"p2p_unavailable": str(e).splitlines()[0][:300]}
    info = plan.info
    total_kv = p.kv_bytes                       # whole job
    local_kv = info.kv_bytes
    stream = torch.cuda.current_stream(dev)
    rows, d = p.batch * p.heads_q, p.head_dim
    nq = (args.q_len,) if args.q_len > 1 else ()
    out = torch.empty(p.batch, p.heads_q, *nq, d, dtype=torch.float32, device=dev)
    lse = torch.empty(p.batch, p.heads_q, *nq, dtype=torch.float32, device=dev)
    if world > 1:   # the NCCL path: O_r and L_r written into ONE packed buffer, ONE all-gather
        packed = torch.empty(rows * (d + 1), dtype=torch.float32, device=dev)
        po, pl = packed[:rows * d].view(rows, d), packed[rows * d:]
        allp = torch.empty(world, rows * (d + 1), dtype=torch.float32, device=dev)
        fin_o = torch.empty(rows, d, dtype=torch.float32, device=dev)
        fin_l = torch.empty(rows, dtype=torch.float32, device=dev)

        def gather_packed():
            if args.backend == "nccl":
                dist.all_gather_into_tensor(allp, packed)
            else:
                allp.copy_(sharded.gather_packed(packed))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if total_kv < 2 * L2_BYTES else None

    def step_single(ev0=None, ev1=None):
        if flush is not None:
            flush.zero_()
        if ev0 is not None:
            ev0.record(stream)
        plan.decode(q, k, v, out, lse, stream=stream)   # fused: the exchange + fold run inside
        if ev1 is not None:
            ev1.record(stream)

    def step_nccl(ev0=None, ev1=None):
        if ev0 is not None:
            ev0.record(stream)
        plan.decode_partial(q, k, v, po, pl, stream=stream)
        if ev1 is not None:
            ev1.record(stream)
        gather_packed()
        la_combine_packed(allp, world, rows, d, fin_o, fin_l, stream=stream)

    def sync():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(*vals):
        if world == 1:
            return list(vals)
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist()

    # SM-rate-weighted stream-K (la_plan_calibrate): a plan-setup step, outside the
    # timed region; single GPU, inputs larger than L2 (a flushed config would calibrate warm)
    weights_note = "equal (Eq. 2)" if SCHEDULE_NAMES[plan.info.schedule] == "streamk" else None
    if args.sm_weights == "calibrate" and SCHEDULE_NAMES[plan.info.schedule] == "streamk" and world == 1 \
            and flush is None:
        plan.calibrate(q, k, v, launches=6, rounds=2, stream=stream)
        rl = plan.range_lengths()
        weights_note = (f"calibrated (la_plan_calibrate: 2 rounds x 6 launches; LeanTiles per CTA "
                        f"{int(rl.min())}..{int(rl.max())})")
    info = plan.info
    paths = {}
    if world > 1:
        for _ in range(args.warmup):
            step_nccl()
        if fused:   # the fused exchange must agree with partial + all-gather + la_combine
            for _ in range(args.warmup):
                step_single()
            sync()
            bad = 0.0
            try:
                plan.xchg_status()
            except la.LaError:
                bad = 1.0
            step_nccl()
            step_single()
            try:
                plan.xchg_status()
            except la.LaError:
                bad = 1.0
            chk = torch.tensor([bad, (out.view(rows, -1) - fin_o).abs().max().item(),
                                (lse.view(rows) - fin_l).abs().max().item()], dtype=torch.float64, device=dev)
            dist.all_reduce(chk, op=dist.ReduceOp.MAX)   # one collective decision for all ranks
            bad, do, dl = chk.tolist()
            xchg_note = {"max_abs_diff_vs_nccl_combine": [do, dl]}
            if bad or max(do, dl) > 1e-5:
                fused = False
                xchg_note["p2p_rejected"] = "exchange wait timed out" if bad else "disagrees with the NCCL combine"
        # time BOTH exchange paths (the north star's NCCL combine and the fused NVLink fixup)
        ms, kern = _timed_loop(step_nccl, args.steps, stream, sync)
        ms, kmean = max_over_ranks(ms, sum(kern) / len(kern))
        paths["nccl_allgather_combine"] = {"step_us": ms * 1e3, "kernel_us": kmean * 1e3}
        if fused:
            ms_f, kern_f = _timed_loop(step_single, args.steps, stream, sync)
            ms_f, kmean_f = max_over_ranks(ms_f, sum(kern_f) / len(kern_f))
            paths["fused_p2p"] = {"step_us": ms_f * 1e3, "kernel_us": kmean_f * 1e3}
    else:
        for _ in range(args.warmup):
            step_single()
    # ---- the timed region of the reported line ------------------------------------------
    # K back-to-back steps between two events (per-launch events only when a step holds other
    # GPU work to exclude -- the L2 flush of small configs -- or an exchange: they add ~5 us
    # per step); the per-launch distribution comes from a second, instrumented pass
    main_step = step_single if (world == 1 or fused) else step_nccl
    per_launch = flush is not None or world > 1
    sync()
    launches0 = la.launch_count()
    with ClockSampler(local) as clk:
        step_ms, kern_each = _timed_loop(main_step, args.steps, stream, sync, per_launch)
    launches = la.launch_count() - launches0
    if kern_each is None:   # one decode launch per step and nothing else: launch time = step time
        kern_ms = step_ms
        _, kern_each = _timed_loop(main_step, args.steps, stream, sync, True)
    else:
        kern_ms = sum(kern_each) / args.steps
    pct = {f"p{q_}": kern_each[min(len(kern_each) - 1, int(q_ / 100 * len(kern_each)))] * 1e3 for q_ in (10, 50, 90)}
    unflushed_us = None
    if flush is not None and world == 1:   # L2-resident config: also the warm-L2 kernel time
        u0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        u1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            u0[i].record(stream)
            plan.decode(q, k, v, out, lse, stream=stream)
            u1[i].record(stream)
        torch.cuda.synchronize(dev)
        unflushed_us = sorted(a.elapsed_time(b) for a, b in zip(u0, u1))[args.steps // 2] * 1e3
    if flush is not None and world == 1:   # the flush is not part of the step: report the kernel time
        step_ms = kern_ms
    step_ms, kern_ms = max_over_ranks(step_ms, kern_ms)

    # ---- N > 1: the same workload unsharded on rank 0's GPU (T_1) -------------------------
    scaling = None
    if world > 1:
        t1_ms = 0.0
        if rank == 0:
            k1 = synth.fill_kv_cache(p, "k", dev)
            v1 = synth.fill_kv_cache(p, "v", dev)
            plan1 = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, **plan_kw)
            o1 = torch.empty_like(out)
            l1 = torch.empty_like(lse)

            def step1(ev0=None, ev1=None):
                if ev0 is not None:
                    ev0.record(stream)
                plan1.decode(q, k1, v1, o1, l1, stream=stream)
                if ev1 is not None:
                    ev1.record(stream)
            for _ in range(args.warmup):
                step1()
            torch.cuda.synchronize(dev)
            t1_ms, _ = _timed_loop(step1, max(3, min(args.steps, 20)), stream, lambda: torch.cuda.synchronize(dev))
            del k1, v1
        (t1_ms,) = max_over_ranks(t1_ms)   # only rank 0 measured: the max is its value
        peak, _ = peaks()
        per_gpu = local_kv / (kern_ms * 1e-3) / 1e9
        scaling = {"t1_us": t1_ms * 1e3, "tp_us": step_ms * 1e3, "scaling_efficiency": t1_ms / (world * step_ms),
                   "per_gpu_gbs": per_gpu, "per_gpu_frac": per_gpu / peak,
                   "per_gpu_kv_bytes": local_kv, "exchange_paths": paths,
                   "note": "T_1 = the unsharded workload on rank 0's GPU in this run; efficiency = T_1 / (P T_P)"}

    # ---- end to end through the C ABI with host buffers ---------------------------------
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        qh = q.cpu().pin_memory()
        kh = k.cpu().pin_memory()
        vh = v.cpu().pin_memory()
        oh = torch.empty(rows * (d + 1), dtype=torch.float32).pin_memory()   # O rows then L (packed)
        ohv, lhv = oh[:rows * d].view(p.batch, p.heads_q, d), oh[rows * d:].view(p.batch, p.heads_q)
        plan.decode_host(qh, kh, vh, ohv, lhv, stream=stream)   # warm-up (allocates staging)
        fin_h = torch.empty(rows, d, dtype=torch.float32).pin_memory()
        sync()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            plan.decode_host(qh, kh, vh, ohv, lhv, stream=stream)
            if world > 1 and not fused:   # the shard result goes through the exchange and the combine
                packed.copy_(oh, non_blocking=True)
                gather_packed()
                la_combine_packed(allp, world, rows, d, fin_o, fin_l, stream=stream)
                fin_h.copy_(fin_o, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        (e2e_ms,) = max_over_ranks(e0.elapsed_time(e1) / args.e2e_steps)
        e2e = {"value": total_kv / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(qh.numel() * qh.element_size() + 2 * kh.numel() * kh.element_size()),
               "d2h_bytes_per_step": int(rows * (d + 1) * 4)}

    # ---- oracle cpu_baseline (rank 0, N = 1 only) -----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        units = oracle_sample(p, min(args.cpu_heads, p.batch * p.heads_kv), device=dev)
        secs = run_oracle_sample(units, p.scale)
        cpu = {"value": sample_bytes(units, synth.DTYPE_BYTES[p.dtype]) / secs / 1e9, "unit": "GB/s",
               "cores": blas_threads(), "host_cores": os.cpu_count(), "kind": "oracle", "seconds": secs,
               "sample": f"{len(units)} of {p.batch * p.heads_kv} (b, h_kv) units of {cfg} (full context each); "
                         f"cores = the numpy/BLAS threads the oracle used, host_cores = the box's logical CPUs"}
        try:   # the same oracle on ONE core, on a smaller bounded sample
            from threadpoolctl import threadpool_limits
            one = units[:max(1, len(units) // 8)]
            with threadpool_limits(1):
                secs1 = run_oracle_sample(one, p.scale)
            cpu["single_thread"] = {"value": sample_bytes(one, synth.DTYPE_BYTES[p.dtype]) / secs1 / 1e9,
                                    "seconds": secs1, "sample": f"{len(one)} unit(s)"}
        except ImportError:
            pass

    if rank == 0:
        peak, peak_src = peaks()
        achieved = local_kv / (kern_ms * 1e-3) / 1e9   # dominant kernel, per launch
        traffic = ncu_traffic(cfg + (f"-q{p.q_len}" if p.q_len > 1 else "") + ("-fp8" if p.dtype == "fp8" else "")
                              + ("-tc5" if info.engine == 1 and info.tile_rows > 1 else ""))
        engine = "Fp8" if p.dtype == "fp8" else (("Tc5" if info.engine == 1 else "Gqa")
                                                 if info.tile_rows > 1 else "Mha")
        line = {
            "metric": METRIC, "value": total_kv / (step_ms * 1e-3) / 1e9, "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
            "latency_us": step_ms * 1e3, "higher_is_better": True,
            "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": p.dtype,
            "data": "synthetic (seeded counter-based generator, distribution D1; DESIGN.md input recipe)",
            "config": {"workload": f"{cfg}: {WORKLOADS[cfg]}" + (
                           f" -- FP8 E4M3 KV variant (k_scale {p.k_scale}, v_scale {p.v_scale}, bf16 q)"
                           if p.dtype == "fp8" else ""), "batch": p.batch, "heads_q": p.heads_q,
                       "heads_kv": p.heads_kv, "head_dim": p.head_dim,
                       "context": p.ctx_lens[0] if len(set(p.ctx_lens)) == 1 else p.ctx_lens,
                       "kv_bytes": total_kv, "tile_n": info.tile_n, "grid": info.grid,
                       "stage_tokens": info.stage_tokens,
                       "schedule": SCHEDULE_NAMES[info.schedule] + (" (auto)" if args.schedule == "auto" else ""),
                       "quantization_efficiency": info.quantization_efficiency,
                       **({"sm_weights": weights_note} if weights_note else {}),
                       **({"engine": {0: "mma.sync", 1: "tcgen05"}[info.engine]} if info.engine >= 0 else {}),
                       **({"q_len": args.q_len, "query_tile_rows": info.tile_rows, "units": info.num_units}
                          if args.q_len > 1 else {}),
                       "kv_layout": p.layout + (f" (page {args.page_size})" if args.page_size else ""),
                       "virtual_ctas": info.num_vctas,
                       "l2": ("inputs > L2 (no flush)" if flush is None else "L2 flushed (512 MB memset) before every step"),
                       "parallelism": "single GPU" if world == 1 else
                       (f"sequence-sharded x{world}, fused in-kernel NVLink exchange (NEXT-2)" if fused else
                        f"sequence-sharded x{world} + {args.backend.upper()} all-gather (one packed O||L message) "
                        f"+ la_combine_strided"),
                       **({"exchange_check": xchg_note} if xchg_note else {})},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": f"la_decode<{engine}Engine<{p.dtype},{p.head_dim}>>", "kernel_us": kern_ms * 1e3,
                         "kernel_us_pct": pct, "kernel_us_pct_note": "per-launch event pairs, separate instrumented pass",
                         **({"kernel_us_unflushed_p50": unflushed_us} if unflushed_us is not None else {}),
                         "algorithmic_bytes_per_launch": local_kv,
                         "read_probe_gbs": read_probe_gbs(),
                         "frac_of_read_probe": (achieved / read_probe_gbs()) if read_probe_gbs() else None},
            **({"multi_gpu": scaling} if scaling else {}),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return bench_reference(args)
    return bench_ours(args)


if __name__ == "__main__":
    sys.exit(main())
