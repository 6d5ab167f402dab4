# LA_TC5_SPLIT=2 (two accumulator chains per contraction) vs default, c3 N_q = 4 / 2; parity on the variant
LEANATTN_LIB=variants/libla_split2.so timeout 500 python -m pytest tests/test_gpu_tcgen05.py -q -x -m gpu -k "wide or tiny" 2>&1 | tail -2
B=variants/libla_split2.so Q=4 bash scripts/tc5_ab.sh
B=variants/libla_split2.so Q=2 bash scripts/tc5_ab.sh
