timeout 600 python -m pytest tests/test_gpu_update.py tests/test_gpu_decode.py tests/test_gpu_graph.py tests/test_gpu_xchg.py -q > gpurun_out/t_dyn.log 2>&1; tail -5 gpurun_out/t_dyn.log
for args in "c2 --schedule dynamic --first 900" "c2 --schedule dynamic --first 960 --min 4" "c2 --schedule dynamic --first 950 --min 4" "c2 --schedule dynamic --first 970 --min 3" "c3 --engine mma --schedule dynamic --min 4" "c3 --engine mma --schedule dynamic --first 900 --min 4" "c3 --engine mma --schedule dynamic --first 900 --min 6" "c3 --engine mma --schedule dynamic --first 850 --min 8" "c3 --engine tcgen05 --schedule dynamic --first 900 --min 6"; do
  timeout 120 python scripts/tail_report.py $args 2>&1 | head -5
done
