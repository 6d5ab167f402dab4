set -x
for args in "c2" "c2 --schedule dynamic" "c2 --schedule dynamic --first 900 --min 4" "c2 --schedule dynamic --first 950 --min 8" "c2 --schedule fixed_split" "c3 --engine mma" "c3 --engine tcgen05" "c3 --engine mma --schedule dynamic --first 950 --min 8" "c4"; do
  timeout 120 python scripts/tail_report.py $args 2>&1 | tail -12
done
