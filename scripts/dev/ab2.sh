V=paper_2405_10480_b200/lib/variants
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_all.log 2>&1; tail -2 gpurun_out/t_all.log
bash scripts/ab_bench.sh "--config c1" $V/r01.so cur
bash scripts/ab_bench.sh "--config c2" $V/r01.so cur
for d in "940 8" "940 4" "950 6" "930 8" "960 4"; do set -- $d; bash scripts/ab_bench.sh "--config c2 --schedule dynamic --dyn-first $1 --dyn-min $2" cur; done
for args in "c2 --schedule dynamic --min 8" "c2 --schedule dynamic --min 4" "c3 --engine mma --schedule dynamic --min 8"; do timeout 120 python scripts/tail_report.py $args 2>&1; done
