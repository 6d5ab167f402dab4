timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -3 gpurun_out/t_all.log
for a in "--schedule streamk" "--schedule dynamic --dyn-first 940 --dyn-min 8" "--schedule dynamic --dyn-first 940 --dyn-min 4" "--schedule dynamic --dyn-first 960 --dyn-min 4"; do
 for c in c2 c4 c3; do
  timeout 300 python bench.py --config $c $a --steps 100 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c $a', round(d['ms_per_step']*1e3,1), 'us/step kernel', round(r['kernel_us'],1), 'p10/50/90', [round(x,1) for x in r['kernel_us_pct'].values()], d['clocks']['sm_mhz'])"
 done
done
timeout 300 python bench.py --config c3 --engine tcgen05 --steps 100 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c3 tc5', round(d['ms_per_step']*1e3,1), 'us/step kernel', round(r['kernel_us'],1))"
timeout 300 python bench.py --config c1 --steps 100 --warmup 5 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('c1', round(d['ms_per_step']*1e3,1), 'us/step kernel', round(r['kernel_us'],1))"
