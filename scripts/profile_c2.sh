# ncu evidence for the c2 north-star run (see /opt/skills/guides/B200_PROFILING.md)
set -x
python -c "import __graft_entry__ as g; g.build()"
# 1) every launch of the bench command with its device time (cold, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/launches_bench.log 2>&1
# 2) one full capture of the top kernel
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:la_decode_mha -s 3 -c 1 \
    -o gpurun_out/prof_c2 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/prof_c2.log 2>&1
ls -la gpurun_out/
