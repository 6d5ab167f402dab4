#!/bin/bash
# Full evaluation pass on one B200 (run under gpurun): smoke, the GPU test suite, the default
# bench line (+ e2e + cpu baseline), the reference arm, every config / engine / schedule
# variant, and ncu evidence (launch list + one full capture) for the main configs.
# Everything lands in gpurun_out/$R/ (R = round tag, default r02).
R=${R:-r02}
O=gpurun_out/$R
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -n 3 $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -n 2 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_c2.json 2> $O/bench_c2.err; tail -c 400 $O/bench_c2.json
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.json 2>&1
run() {  # name, bench args
  timeout 600 python bench.py $2 --no-cpu --no-e2e > $O/bench_$1.json 2> $O/bench_$1.err
  python -c "import json,sys; d=json.loads(open('$O/bench_$1.json').read().strip().splitlines()[-1]); r=d['roofline']; print('%-14s %8.1f us/step  kernel p50 %7.1f  %6.0f GB/s  frac %.3f  %s' % ('$1', d['ms_per_step']*1e3, r['kernel_us_pct']['p50'], r['achieved'], r['frac'], d['config'].get('schedule')))" 2>/dev/null || echo "$1 failed"
}
run c1 "--config c1"
run c2_streamk "--config c2 --schedule streamk"
run c3 "--config c3"
run c3_mma "--config c3 --engine mma"
run c3_cal "--config c3 --sm-weights calibrate"
run c3_mma_cal "--config c3 --engine mma --sm-weights calibrate"
run c3_q2 "--config c3 --q-len 2"
run c3_q4 "--config c3 --q-len 4"
run c4 "--config c4"
run c4_streamk "--config c4 --schedule streamk"

run c5 "--config c5"
run c2_fp8 "--config c2 --dtype fp8"
run c3_fp8 "--config c3 --dtype fp8"
run c2_paged16 "--config c2 --page-size 16"
run c3_paged16 "--config c3 --page-size 16"
run c3_paged16_tc5 "--config c3 --page-size 16 --engine tcgen05"
for cfg in "c2|--config c2|c2" "c3|--config c3|c3-tc5" "c3_mma|--config c3 --engine mma|c3" "c4|--config c4|c4" "c1|--config c1|c1" "c3_q4|--config c3 --q-len 4|c3-q4-tc5" "c3_q2|--config c3 --q-len 2|c3-q2-tc5"; do
  IFS='|' read -r name args key <<< "$cfg"
  bash scripts/profile.sh ${R}_$name "$args" $key > $O/profile_$name.log 2>&1
  mv gpurun_out/${R}_${name}* $O/ 2>/dev/null
done
ls -la $O | tail -40
