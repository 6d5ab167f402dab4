# smoke (incl. FP8), fused-exchange tests, ncu captures of the FP8 defaults (c2, c3)
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_xchg.py tests/test_gpu_fp8.py -q -x 2>&1 | tail -3
for c in c2 c3; do
  timeout 300 python bench.py --config $c --dtype fp8 --no-cpu --no-e2e > gpurun_out/bench_${c}_fp8.json 2>&1; tail -c 300 gpurun_out/bench_${c}_fp8.json; echo
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_${c}_fp8 python bench.py --config $c --dtype fp8 --steps 5 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_c2_fp8.csv python bench.py --dtype fp8 --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ls gpurun_out
