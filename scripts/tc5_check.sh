# tcgen05 engine: parity tests, then c3 timing on both engines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_tcgen05.py -x -q > gpurun_out/tc5_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 30 gpurun_out/tc5_pytest.log
for e in tcgen05 mma; do
  timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu --no-e2e --engine $e > gpurun_out/tc5_bench_c3_$e.json 2>&1; tail -c 700 gpurun_out/tc5_bench_c3_$e.json; echo
done
