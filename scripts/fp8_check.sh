# FP8 KV (NEXT-4) on one B200: build, parity tests, a regression subset, bench c2/c3 in fp8.
set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fp8_build.log 2>&1 || tail -20 gpurun_out/fp8_build.log
timeout 900 python -m pytest tests/test_gpu_fp8.py -q -x > gpurun_out/fp8_pytest.log 2>&1; tail -15 gpurun_out/fp8_pytest.log
timeout 900 python -m pytest tests -m gpu -q -x -k "not fp8" > gpurun_out/fp8_regress.log 2>&1; tail -3 gpurun_out/fp8_regress.log
for c in c2 c3 c4; do
  timeout 300 python bench.py --config $c --dtype fp8 --no-cpu --no-e2e > gpurun_out/bench_${c}_fp8.json 2>&1; tail -c 1200 gpurun_out/bench_${c}_fp8.json
done
timeout 300 python bench.py --config c3 --dtype fp8 --page-size 16 --no-cpu --no-e2e > gpurun_out/bench_c3_fp8_p16.json 2>&1; tail -c 600 gpurun_out/bench_c3_fp8_p16.json
