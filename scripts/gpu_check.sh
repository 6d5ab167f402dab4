set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -6
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
for s in dynamic streamk; do
  timeout 300 python bench.py --steps 300 --warmup 10 --no-cpu --no-e2e --schedule $s 2>&1 | tail -1
  timeout 300 python bench.py --config c3 --steps 300 --warmup 10 --no-cpu --no-e2e --schedule $s 2>&1 | tail -1
  timeout 300 python bench.py --config c4 --steps 100 --warmup 5 --no-cpu --no-e2e --schedule $s 2>&1 | tail -1
  python scripts/trace_c2.py c2 $s 2>&1 | tail -6
done
