set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -5
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30
timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu 2>&1 | tail -3
