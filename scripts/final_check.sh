# End-of-round check at HEAD: smoke, the whole GPU suite, the default bench line and the c3 engine benches
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 2 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 300 gpurun_out/bench_default.json
timeout 300 python bench.py --config c3 --engine tcgen05 --no-cpu --no-e2e > gpurun_out/bench_c3_tc5.json 2>&1
for ql in 2 4; do for e in auto mma; do timeout 300 python bench.py --config c3 --q-len $ql --engine $e --no-cpu --no-e2e > gpurun_out/bench_c3_q${ql}_$e.json 2>&1; done; done
for f in gpurun_out/bench_c3*.json; do echo $f; tail -c 200 $f; echo; done
