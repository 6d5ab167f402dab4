python -c "import __graft_entry__ as g; g.build()"
r() { timeout 300 python bench.py "$@" --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['kernel_us'],2), 'us', round(d['roofline']['achieved']), 'GB/s', d['clocks']['sm_mhz'])"; }
r --config c1
r --config c1 --schedule dynamic
for c in c2 c4; do
  r --config $c
  for f in 950 970 985; do for m in 4 8; do r --config $c --schedule dynamic --dyn-first $f --dyn-min $m; done; done
  r --config $c
done
