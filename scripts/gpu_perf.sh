# quick perf comparison of the schedules (no tests)
python -c "import __graft_entry__ as g; g.build()"
for c in c2 c3 c4; do
  for s in "streamk" "dynamic --dyn-first 750 --dyn-min 2" "dynamic --dyn-first 850 --dyn-min 4" "dynamic --dyn-first 920 --dyn-min 8"; do
    timeout 300 python bench.py --config $c --steps 200 --warmup 10 --no-cpu --no-e2e --schedule $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$s', round(d['latency_us'],1), 'us', round(d['value']), 'GB/s', d['config'].get('virtual_ctas'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
python scripts/trace_c2.py c2 dynamic 2>&1 | tail -9
