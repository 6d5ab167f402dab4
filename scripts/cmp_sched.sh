# static vs dynamic schedule on the bench configs (kernel time, 3 alternating repeats)
python -c "import __graft_entry__ as g; g.build()"
r() { timeout 300 python bench.py "$@" --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['kernel_us'],1), 'us', round(d['roofline']['achieved']), 'GB/s', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1; do
for c in c2 c3 c4; do
  r --config $c
  r --config $c --schedule dynamic
  r --config $c --schedule dynamic --dyn-first 900 --dyn-min 4
done
done
