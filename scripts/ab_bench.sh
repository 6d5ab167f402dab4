#!/bin/bash
# Same-box A/B timing of library variants: ab_bench.sh "<bench args>" lib1.so lib2.so ...  (lib "cur" = in-tree)
# Two alternating rounds per variant; prints us/step and kernel p50 per run.
ARGS=$1; shift
for round in 1 2; do
  for lib in "$@"; do
    if [ "$lib" = "cur" ]; then L=""; else L="LEANATTN_LIB=$lib"; fi
    env $L timeout 300 python bench.py $ARGS --steps 100 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('%-40s %-28s %8.1f us/step  kernel p50 %7.1f  clk %s' % ('$ARGS', '$(basename $lib)', d['ms_per_step']*1e3, r['kernel_us_pct']['p50'], d['clocks']['sm_mhz']))"
  done
done
