# paged KV (NEXT-4) cost vs the contiguous layout, MHA c2 and GQA c3
python -c "import __graft_entry__ as g; g.build()"
r() { timeout 300 python bench.py "$@" --steps 100 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['roofline']['kernel_us'],1), 'us', round(d['roofline']['achieved']), 'GB/s')"; }
for c in c3 c2; do
  r --config $c
  for ps in 16 32 64 256; do r --config $c --page-size $ps; done
done
