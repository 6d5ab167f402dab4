# tcgen05 engine: NWG warpgroups over an NST-slot ring -- parity + c3 timings (default lib, then a variant)
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -q -x -m gpu 2>&1 | tail -2
for q in 4 2; do timeout 120 python bench.py --config c3 --q-len $q --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("default q'$q'", d["ms_per_step"], d["value"])'; done
export LEANATTN_LIB=variants/libla_nwg16.so
timeout 400 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -q -x -m gpu 2>&1 | tail -2
for q in 2; do timeout 120 python bench.py --config c3 --q-len $q --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("nwg16=2 q'$q'", d["ms_per_step"], d["value"])'; done
