# c1 (latency-bound) sweep over LeanTile size and schedule.
python -c "import __graft_entry__ as g; g.build()"
r() { timeout 300 python bench.py "$@" --steps 300 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['kernel_us'],2), 'us', d['clocks']['sm_mhz'])"; }
for rep in 1; do
for t in 0 32 64 128 256; do
  r --config c1 --tile-n $t
  r --config c1 --tile-n $t --schedule dynamic
  r --config c1 --tile-n $t --schedule fixed_split
done
r --config c1 --schedule sequential
done
