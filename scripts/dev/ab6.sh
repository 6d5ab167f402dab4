for r in 1 2 3; do
for c in "--config c4" "--config c4 --schedule streamk" "--config c2" "--config c2 --schedule streamk"; do
  bash scripts/ab_bench.sh "$c" cur 2>&1 | head -1
done; done
timeout 120 python scripts/tail_report.py c4 --schedule dynamic 2>&1 | head -7
timeout 120 python scripts/tail_report.py c4 2>&1 | head -7
