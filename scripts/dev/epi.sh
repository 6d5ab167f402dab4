V=paper_2405_10480_b200/lib/variants
for args in "c3 --engine mma --schedule dynamic --min 4" "c3 --engine mma --schedule dynamic --min 8" "c2 --schedule dynamic --min 8"; do LA_EPI_TRACE=1 LEANATTN_LIB=$V/epitrace.so timeout 120 python scripts/tail_report.py $args 2>&1 | head -8; done
bash scripts/ab_bench.sh "--config c1" $V/r01.so cur
