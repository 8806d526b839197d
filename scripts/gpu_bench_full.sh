set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -4 gpurun_out/bench.log
KR='regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --csv --log-file gpurun_out/launches_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 5 --sparse-only > /dev/null 2> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:sp_gemm|sp_potrf|apply_kernel' -s 200 -c 6 -o gpurun_out/prof_c3_sparse python bench.py --steps 1 --warmup 3 --applies 3 --sparse-only > /dev/null 2> gpurun_out/ncu_full.log
ls gpurun_out
