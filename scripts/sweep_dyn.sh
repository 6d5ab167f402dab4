python -c "import __graft_entry__ as g; g.build()"
for c in c2 c3 c4; do
  for f in 750 850 920; do
    for m in 2 4 8; do
      timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --no-e2e --schedule dynamic --dyn-first $f --dyn-min $m 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c f=$f m=$m', round(d['latency_us'],1), 'us', round(d['value']), 'GB/s vctas', d['config'].get('virtual_ctas'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
    done
  done
  timeout 300 python bench.py --config $c --steps 100 --warmup 5 --no-cpu --no-e2e --schedule streamk 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c streamk', round(d['latency_us'],1), 'us', round(d['value']), 'GB/s')"
done
