python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -4
for c in c2 c3 c4; do
  for s in "streamk"; do
    timeout 300 python bench.py --config $c --steps 300 --warmup 10 --no-cpu --no-e2e --schedule $s 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$s', round(d['latency_us'],1), 'us', round(d['value']), 'GB/s kernel', round(d['roofline']['kernel_us'],1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
