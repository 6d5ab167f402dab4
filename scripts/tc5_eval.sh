mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; tail -n 3 gpurun_out/pytest_gpu.log
b() {
  LEANATTN_LIB=$3 timeout 300 python bench.py --config c3 --steps 300 --warmup 10 --no-cpu --no-e2e --engine $2 > gpurun_out/tc5_bench_$1.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/tc5_bench_$1.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$1', round(r['kernel_us'],1), 'us', round(r['achieved']), 'GB/s', r['kernel_us_pct'])"
}
b tc5 tcgen05
b tc5_split2 tcgen05 $PWD/paper_2405_10480_b200/lib/v/split2.so
b mma mma
b tc5b tcgen05
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c3_tc5 python bench.py --config c3 --engine tcgen05 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c3_tc5.log 2>&1
echo done
