# Round-2 final evidence on the final code (k-slice skipping): full GPU suite, smoke, bench lines, launch list.
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02j_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r02j_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02j_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r02j_bench_c3.json 2> gpurun_out/r02j_bench_c3.err; echo "c3 exit $?"
timeout 900 python bench.py --config c4 --no-cpu-baseline > gpurun_out/r02j_bench_c4.json 2> gpurun_out/r02j_bench_c4.err; echo "c4 exit $?"
timeout 1200 python bench.py --config c5 --no-cpu-baseline > gpurun_out/r02j_bench_c5.json 2> gpurun_out/r02j_bench_c5.err; echo "c5 exit $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel' --csv \
  --log-file gpurun_out/r02j_c3_launches.csv python scripts/factor_bench.py c3 1 > gpurun_out/r02j_ncu1.log 2>&1
echo "ncu exit $?"
