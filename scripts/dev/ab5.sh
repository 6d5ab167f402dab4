V=paper_2405_10480_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
for c in "--config c2" "--config c2 --schedule streamk" "--config c4" "--config c4 --schedule streamk" "--config c2 --dtype fp8" "--config c2 --dtype fp8 --schedule streamk" "--config c3 --engine tcgen05 --schedule dynamic --dyn-min 8" "--config c3 --engine tcgen05 --schedule dynamic --dyn-min 4" "--config c3 --engine tcgen05" "--config c3" "--config c5" "--config c5 --schedule streamk"; do
  bash scripts/ab_bench.sh "$c" cur 2>&1 | head -1
done
