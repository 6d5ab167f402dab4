# static (Alg. 2) vs dynamic schedule on c2/c3/c4, bf16 and fp8.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for dt in bf16 fp8; do for c in c2 c3 c4; do for s in streamk dynamic; do
  timeout 300 python bench.py --config $c --dtype $dt --schedule $s --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$dt', '$c', '$s', round(r['kernel_us'],1), 'us p10/p50/p90', [round(x,1) for x in r['kernel_us_pct'].values()], round(r['achieved']), 'GB/s', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done; done
