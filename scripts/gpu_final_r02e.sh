# Round-2 evidence on the final code (part 1): sanitizers over every kernel
# family (incl. the trsm path, implicit sparse route, device solve_local),
# the ncu launch list of a c3 step and full sets of the changed tail kernels.
set -x
rm -f gpurun_out/sanitize_summary.txt
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/r02e_sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel' --csv \
  --log-file gpurun_out/r02e_c3_launches.csv python scripts/factor_bench.py c3 1 > gpurun_out/r02e_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:syrk_kernel|sp_u2' -s 2 -c 2 \
  -o gpurun_out/r02e_tail python scripts/factor_bench.py c3 1 > gpurun_out/r02e_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:implicit_apply' -s 10 -c 1 \
  -o gpurun_out/r02e_implicit python scripts/implicit_bench.py c3 10 > gpurun_out/r02e_ncu3.log 2>&1
python scripts/sass_summary.py > gpurun_out/r02e_sass.md
ls -la gpurun_out | tail -20
