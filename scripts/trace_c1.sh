python -c "import __graft_entry__ as g; g.build()"
for a in "streamk 256" "streamk 32" "dynamic 256" "fixed_split 256" "streamk 64"; do
  timeout 120 python scripts/trace_case.py c1 $a 2>&1 | head -140
done
