# racecheck for one engine's cases, every hazard aggregated by (access site pair) -- the raw
# log is too large to keep.   bash scripts/racecheck_summary.sh tcgen05
mkdir -p gpurun_out
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 1000000 python scripts/sanitize_case.py $1 2>&1 \
 | grep -E "^=========     (Read|Write) Thread|RACECHECK SUMMARY|sanitize case" \
 | sed -E 's/Thread \([0-9]+,0,0\)//; s/la::<unnamed>:://g; s/\(la::DecodeArgs, la::TmapPair\)//; s/\+0x[0-9a-f]+//; s/\(la::[^)]*\)//g; s/\([^()]*State &[^)]*\)//' \
 | sort | uniq -c | sort -rn > gpurun_out/racecheck_summary_$1.txt
cat gpurun_out/racecheck_summary_$1.txt | head -30
