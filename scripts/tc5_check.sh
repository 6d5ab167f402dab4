# tcgen05 engine: parity tests, then c3 timing (default build + variants under lib/v/)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tcgen05.py -x -q > gpurun_out/tc5_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/tc5_pytest.log
b() {  # label, engine, [lib]
  LEANATTN_LIB=$3 timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu --no-e2e --engine $2 > gpurun_out/tc5_bench_$1.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/tc5_bench_$1.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(r['kernel_us'],1), 'us', round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'])"
}
b tc5 tcgen05
b mma mma
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/tc5_bench_c2.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/tc5_bench_c2.json').read().strip().splitlines()[-1]); r=d['roofline']; print('c2 mha', round(r['kernel_us'],1), 'us', round(r['achieved']), 'GB/s')"
for v in paper_2405_10480_b200/lib/v/*.so; do b tc5_$(basename $v .so) tcgen05 $PWD/$v; done
timeout 120 python scripts/trace_tail.py c3 tcgen05 2>&1 | head -4
