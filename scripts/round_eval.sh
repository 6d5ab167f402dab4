# Full evaluation pass on one B200: build, smoke, GPU tests, bench (+e2e, +cpu baseline),
# reference arm, other configs / engines, ncu launch list + full captures.
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -n 5 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -n 3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; tail -c 2500 gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_reference.json 2>&1; tail -c 600 gpurun_out/bench_reference.json
for c in c3 c4; do timeout 300 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_$c.json 2>&1; done
timeout 300 python bench.py --config c3 --engine tcgen05 --no-cpu --no-e2e > gpurun_out/bench_c3_tc5.json 2>&1
for ql in 2 4; do for e in auto mma; do timeout 300 python bench.py --config c3 --q-len $ql --engine $e --no-cpu --no-e2e > gpurun_out/bench_c3_q${ql}_$e.json 2>&1; done; done
for c in c2 c3; do timeout 300 python bench.py --config $c --dtype fp8 --no-cpu --no-e2e > gpurun_out/bench_${c}_fp8.json 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c3 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c3_tc5 python bench.py --config c3 --engine tcgen05 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c3_tc5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c3_q2_tc5 python bench.py --config c3 --q-len 2 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c3_q2_tc5.log 2>&1
ls -la gpurun_out
