# finite initial running max in the tcgen05 engine: parity, then A/B vs the previous build
timeout 500 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -q -x -m gpu 2>&1 | tail -2
B=variants/libla_head.so Q=4 bash scripts/tc5_ab.sh
B=variants/libla_head.so Q=2 bash scripts/tc5_ab.sh
