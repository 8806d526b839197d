# Round-2 evidence on the final code: sanitizers, ncu launch list + full sets,
# a 2-rank (time-shared GPU) bench through the fused exchange, the reference arm.
set -x
rm -f gpurun_out/sanitize_summary.txt
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize.py > gpurun_out/r02_sanitize_$tool.log 2>&1
  echo "$tool exit $?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel' --csv \
  --log-file gpurun_out/r02c_c3_launches.csv python scripts/factor_bench.py c3 1 > gpurun_out/r02c_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:sp_gemm8' -s 300 -c 2 \
  -o gpurun_out/r02c_gemm python scripts/factor_bench.py c3 1 > gpurun_out/r02c_ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:sp_potrf' -s 100 -c 1 \
  -o gpurun_out/r02c_potrf python scripts/factor_bench.py c3 1 > gpurun_out/r02c_ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:trsm_chain|syrk_kernel' -s 2 -c 2 \
  -o gpurun_out/r02c_trsm_syrk python scripts/factor_bench.py c3 1 > gpurun_out/r02c_ncu4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:apply_kernel|reduce_kernel' -s 20 -c 2 \
  -o gpurun_out/r02c_apply python scripts/apply_bench.py c3 20 > gpurun_out/r02c_ncu5.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:pcpg_iter' -s 20 -c 1 \
  -o gpurun_out/r02c_pcpg python scripts/pcpg_bench.py c3 > gpurun_out/r02c_ncu6.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --sparse-only --no-cpu-baseline --no-solve --steps 3 --warmup 3 \
  > gpurun_out/r02_bench_c3_2rank_gloo_1gpu.json 2> gpurun_out/r02_bench_2rank.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_c3_reference_arm.json \
  2> gpurun_out/r02_bench_ref.err
python scripts/sass_summary.py > gpurun_out/r02_sass.md
ls -la gpurun_out
