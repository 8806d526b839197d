set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c3_rcm.json 2> gpurun_out/bench_c3_rcm.log
python bench.py --steps 5 --warmup 3 --ordering interface_last --no-cpu-baseline > gpurun_out/bench_c3_il.json 2> gpurun_out/bench_c3_il.log
KR='regex:unpack_dense|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --csv --log-file gpurun_out/launches_c3_rcm.csv python bench.py --steps 1 --warmup 3 --applies 5 --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:trsm_chain|apply_kernel|block_scale|syrk_kernel|unpack_dense' -s 0 -c 5 -o gpurun_out/prof_c3_rcm python bench.py --steps 1 --warmup 3 --applies 3 --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_full.log
ls -la gpurun_out
