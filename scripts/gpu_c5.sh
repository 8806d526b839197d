set -x
python bench.py --config c5 --steps 3 --warmup 3 --applies 100 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log
tail -5 gpurun_out/bench_c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel' --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --applies 3 --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_c5_launch.log
tail -3 gpurun_out/ncu_c5_launch.log
