set -x
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
  tail -4 gpurun_out/sanitize_$tool.log
done
cat gpurun_out/sanitize_summary.txt
