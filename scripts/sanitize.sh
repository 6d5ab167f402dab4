mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; tail -n 4 gpurun_out/sanitize_$tool.log
done
