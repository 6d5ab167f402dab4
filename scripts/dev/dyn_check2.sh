for args in "c3 --engine mma --schedule dynamic --first 1000" "c3 --engine mma --schedule dynamic --first 900 --min 16" "c3 --engine mma --schedule dynamic --first 850 --min 12" "c2 --schedule dynamic --first 1000" "c2 --schedule dynamic --first 940 --min 8" "c3 --engine mma --schedule streamk"; do
  timeout 120 python scripts/tail_report.py $args 2>&1 | head -5
done
