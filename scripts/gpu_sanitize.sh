set -x
rm -f gpurun_out/sanitize_summary.txt
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
