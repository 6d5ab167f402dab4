mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 7 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 15 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c3 --q-len 2 --steps 200 --warmup 10 --no-cpu --no-e2e > gpurun_out/bench_c3_q2_auto.json 2>&1; tail -c 900 gpurun_out/bench_c3_q2_auto.json
