# tcgen05 16/32-row tiles: parity tests, then c3 (N_q = 1, 2, 4) on both engines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -x -q > gpurun_out/tc5_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 15 gpurun_out/tc5_pytest.log
for ql in 1 2 4; do for e in auto mma; do
  timeout 300 python bench.py --config c3 --q-len $ql --steps 100 --warmup 10 --no-cpu --no-e2e --engine $e > gpurun_out/tc5w_c3_q${ql}_$e.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/tc5w_c3_q${ql}_$e.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c3 q_len $ql $e', r['kernel'], round(r['kernel_us'],1), 'us', round(d['value']), 'GB/s (KV once)', d['config'].get('units'))" 2>&1 | tail -1
done; done
