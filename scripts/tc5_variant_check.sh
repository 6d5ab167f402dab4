mkdir -p gpurun_out
for ql in 4 2; do
python bench.py --config c3 --q-len $ql --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("A q'$ql'", d["ms_per_step"], d["value"])'
LEANATTN_LIB=variants/libla_nst2.so python bench.py --config c3 --q-len $ql --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("B q'$ql'", d["ms_per_step"], d["value"])'
done
python bench.py --config c3 --engine tcgen05 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("A c3 tc5", d["ms_per_step"], d["value"])'
timeout 900 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -q -x -m gpu 2>&1 | tail -3
LEANATTN_LIB=variants/libla_nst2.so timeout 900 python -m pytest tests/test_gpu_tiles.py -q -x -m gpu -k "tcgen05 or 32 or 24" 2>&1 | tail -3
