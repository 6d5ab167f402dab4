mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/hc_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/hc_smoke.log 2>&1; tail -3 gpurun_out/hc_smoke.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/hc_pytest.log 2>&1; tail -3 gpurun_out/hc_pytest.log
timeout 600 python bench.py > gpurun_out/hc_bench.json 2> gpurun_out/hc_bench.err; tail -c 3000 gpurun_out/hc_bench.json
for c in c3; do timeout 300 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/hc_bench_$c.json 2>&1; tail -c 600 gpurun_out/hc_bench_$c.json; done
