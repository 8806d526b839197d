# Round-2 profiles (one GPU, never multi-rank under ncu).  Outputs in gpurun_out/.
set -x
# 1. launch list + per-launch DRAM bytes of one c3 sparse-route step (factorization,
#    assembly, correction) and of the applies (factor_bench: 3 preprocess + 1 resident step)
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel' --csv \
  --log-file gpurun_out/r02_c3_launches.csv python scripts/factor_bench.py c3 1 > gpurun_out/r02_ncu1.log 2>&1
# 2. apply kernels at c3 and c4: duration + DRAM bytes per launch
for c in c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k 'regex:apply_kernel|reduce_kernel' -s 20 -c 10 --csv --log-file gpurun_out/r02_${c}_apply.csv \
    python scripts/apply_bench.py $c 20 > gpurun_out/r02_ncu_apply_$c.log 2>&1
done
# 3. --set full: one launch each of the hot kernels (c3)
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:sp_gemm8|sp_potrf|trsm_chain|syrk_kernel' \
  -s 400 -c 6 -o gpurun_out/r02_c3_full python scripts/factor_bench.py c3 1 > gpurun_out/r02_ncu3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:apply_kernel|pcpg_iter_coop' -s 20 -c 3 \
  -o gpurun_out/r02_c3_apply_full python scripts/pcpg_bench.py c3 > gpurun_out/r02_ncu4.log 2>&1
ls -la gpurun_out/
# 5. PCPG iteration kernels at c3 and c4 (durations per launch)
for c in c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:apply_kernel|pcpg_' -s 300 -c 40 --csv \
    --log-file gpurun_out/r02_${c}_pcpg.csv python scripts/pcpg_bench.py $c > gpurun_out/r02_ncu_pcpg_$c.log 2>&1
done
python scripts/sass_summary.py > gpurun_out/r02_sass.md
