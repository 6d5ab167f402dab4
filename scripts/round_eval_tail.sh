mkdir -p gpurun_out
for c in c3 c4; do timeout 200 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_$c.json 2>&1; done
for ql in 2 4; do timeout 200 python bench.py --config c3 --q-len $ql --engine auto --no-cpu --no-e2e > gpurun_out/bench_c3_q${ql}_auto.json 2>&1; done
for c in c2 c3; do timeout 200 python bench.py --config $c --dtype fp8 --no-cpu --no-e2e > gpurun_out/bench_${c}_fp8.json 2>&1; done
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c2 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c2.log 2>&1
ls -la gpurun_out
