# S^T pre-issue: tcgen05 parity tests, then A/B (default vs LA_TC5_PRES=0) at c3 N_q = 4 and 2
timeout 400 python -m pytest tests/test_gpu_tcgen05.py tests/test_gpu_tiles.py -q -x -m gpu 2>&1 | tail -3
B=variants/libla_nopres.so Q=4 bash scripts/tc5_ab.sh
B=variants/libla_nopres.so Q=2 bash scripts/tc5_ab.sh
