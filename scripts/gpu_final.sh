# Round-end evidence: GPU tests, smoke, default bench (c3), c4/c5 sparse route,
# reference arm, launch list, ncu --set full and DRAM traffic of the factorization
set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log
python bench.py --config c4 --steps 3 --warmup 3 --sparse-only --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel' --csv --log-file gpurun_out/launches_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 5 --sparse-only --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.log
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:sp_gemm8|sp_potrf' --csv --log-file gpurun_out/traffic_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 3 --sparse-only --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_traffic.log
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:sp_gemm8|sp_potrf|apply_kernel|trsm_chain|syrk_kernel' -s 300 -c 8 -o gpurun_out/prof_c3_sparse python bench.py --steps 1 --warmup 3 --applies 3 --sparse-only --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_full.log
ls gpurun_out
