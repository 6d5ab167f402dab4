# dynamic-schedule parameters on GQA c3 (bf16 and fp8)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for dt in bf16 fp8; do for fm in "900 8" "900 16" "950 16" "950 32" "970 32" "850 16"; do set -- $fm
  timeout 300 python bench.py --config c3 --dtype $dt --schedule dynamic --dyn-first $1 --dyn-min $2 --steps 200 --warmup 10 --no-cpu --no-e2e 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$dt', 'first=$1 min=$2', d['config']['virtual_ctas'], round(r['kernel_us'],1), 'us p10/p50/p90', [round(x,1) for x in r['kernel_us_pct'].values()], round(r['achieved']), 'GB/s')"
done; done
