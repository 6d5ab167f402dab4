# tcgen05 engine quick check: parity tests + c3 benches at N_q = 1 / 2 / 4 (+ optional ncu of N_q = 4)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -q -x -m gpu 2>&1 | tail -2
for ql in 4 2 1; do
python bench.py --config c3 --q-len $ql --engine tcgen05 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("c3 tcgen05 q'$ql'", d["ms_per_step"], d["value"])'
done
if [ "$1" = ncu ]; then
timeout 800 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 -o gpurun_out/prof_c3_q4_tc5 python bench.py --config c3 --q-len 4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c3_q4_tc5.log 2>&1
fi
