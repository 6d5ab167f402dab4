#!/bin/bash
# ncu evidence for one bench configuration (see /opt/skills/guides/B200_PROFILING.md):
#   scripts/profile.sh NAME "<bench args>" [KEY]      e.g. scripts/profile.sh r02_c4 "--config c4" c4
# 1) the launch list of the bench command's library kernels (gpu__time_duration per launch: cold, serialised --
#    compare SHARES of the step, not absolutes); 2) one `--set full` capture of the decode kernel;
# 3) the summary into profiles/ncu_summary.json[KEY] + profiles/<NAME>_ncu.md (scripts/ncu_summary.py).
# Run on a GPU box under gpurun; never time anything under ncu.
NAME=$1; ARGS=$2; KEY=${3:-$NAME}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"la_decode|la_combine" -c 60 --csv \
    --log-file gpurun_out/${NAME}_launches.csv python bench.py $ARGS --steps 20 --warmup 3 --no-cpu --no-e2e \
    > gpurun_out/${NAME}_launches.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:la_decode -s 3 -c 1 \
    -o gpurun_out/${NAME} python bench.py $ARGS --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/${NAME}_full.log 2>&1
# summarise locally after gpurun merges gpurun_out/ back (ncu -i needs no GPU):
#   python scripts/ncu_summary.py "$KEY" gpurun_out/${NAME}.ncu-rep gpurun_out/${NAME}_launches.csv --out-md profiles/${NAME}_ncu.md
