# Bench lines (c3 default, c4, c5) on the face ordering + fused graph, and the ncu launch list
# of a c3 step with per-launch DRAM traffic.
set -x
timeout 900 python bench.py > gpurun_out/r02g_bench_c3.json 2> gpurun_out/r02g_bench_c3.err; echo "c3 exit $?"
timeout 900 python bench.py --config c4 > gpurun_out/r02g_bench_c4.json 2> gpurun_out/r02g_bench_c4.err; echo "c4 exit $?"
timeout 1200 python bench.py --config c5 > gpurun_out/r02g_bench_c5.json 2> gpurun_out/r02g_bench_c5.err; echo "c5 exit $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel' --csv \
  --log-file gpurun_out/r02g_c3_launches.csv python scripts/factor_bench.py c3 1 > gpurun_out/r02g_ncu1.log 2>&1
echo "ncu exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:sp_gemm8' -s 300 -c 2 \
  -o gpurun_out/r02g_gemm python scripts/factor_bench.py c3 1 > gpurun_out/r02g_ncu2.log 2>&1
echo "ncu2 exit $?"
ls -la gpurun_out | tail
