"""SM-rate-weighted stream-K: stream-end spread and back-to-back launch time before
and after each la_plan_calibrate round.

  python scripts/calibration_trace.py c3 mma [Q_LEN]
"""
import sys
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import numpy as np, torch, synth, paper_2405_10480_b200 as la
cfg, engine = sys.argv[1], sys.argv[2]
qlen = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = synth.config(cfg, **(dict(q_len=qlen) if qlen > 1 else {}))
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, p.head_dim, p.ctx_lens, trace=True, engine=engine, schedule="streamk", q_len=qlen)
def run(tag, n=5):
    S, E = [], []
    for _ in range(n):
        for _ in range(3): plan.decode(q, k, v)
        torch.cuda.synchronize()
        tr = plan.trace().astype(np.int64)
        t0 = tr[:, 1].min()
        S.append((tr[:, 6] - t0) / 1e3); E.append((tr[:, 5] - t0) / 1e3)
    S = np.array(S); E = np.array(E)
    rl = plan.range_lengths()
    s = S.mean(0); e = E.max(1)
    ev = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): plan.decode(q, k, v)
        e1.record(); torch.cuda.synchronize(); ev.append(e0.elapsed_time(e1) / 20 * 1e3)
    print(f"{cfg} {engine} q{qlen} {tag}: stream_end min/med/max {s.min():.1f}/{np.median(s):.1f}/{s.max():.1f}"
          f"  span(max end) per sample {np.round(e,1)}  tiles {rl.min()}..{rl.max()}  back-to-back us/launch {np.round(ev,1)}")
run("equal")
for rnd in range(3):
    plan.calibrate(q, k, v, launches=4, rounds=1)
    run(f"cal{rnd+1}")
