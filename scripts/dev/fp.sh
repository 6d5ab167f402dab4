cat > /tmp/fp.py <<'PY'
import sys; sys.path.insert(0, "/root/repo")
import torch, synth, paper_2405_10480_b200 as la
p = synth.config("c3")
q, k, v = synth.gen_q(p, "cuda"), synth.fill_kv_cache(p, "k", "cuda"), synth.fill_kv_cache(p, "v", "cuda")
plan = la.Plan(p.batch, p.heads_q, p.heads_kv, 128, p.ctx_lens, schedule="dynamic", dyn_min_chunk=4, engine="mma")
for i in range(3): plan.decode(q, k, v)
torch.cuda.synchronize()
PY
LEANATTN_LIB=paper_2405_10480_b200/lib/variants/foldprint.so python /tmp/fp.py > gpurun_out/fp.log 2>&1; tail -70 gpurun_out/fp.log | sort -t' ' -k14 -n | tail -25
