set -x
rm -f gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel' --csv --log-file gpurun_out/launches_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 5 --sparse-only > gpurun_out/ncu_launch.out 2> gpurun_out/ncu_launch.log
wc -l gpurun_out/launches_c3_sparse.csv
