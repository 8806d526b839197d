# Round-2 final evidence (face ordering + fused step graph): full GPU suite, smoke, the c3 bench line,
# compute-sanitizer over every kernel family.
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02h_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r02h_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r02h_bench_c3.json 2> gpurun_out/r02h_bench_c3.err; echo "bench exit $?"
rm -f gpurun_out/r02h_sanitize_summary.txt
for tool in memcheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/r02h_sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/r02h_sanitize_summary.txt
done
cat gpurun_out/r02h_sanitize_summary.txt
