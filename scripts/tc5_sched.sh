for s in dynamic streamk; do for e in tcgen05 mma; do
 timeout 300 python bench.py --config c3 --steps 200 --warmup 10 --no-cpu --no-e2e --engine $e --schedule $s 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$e $s', round(r['kernel_us'],1), 'us', round(r['achieved']), 'GB/s')"
done; done
