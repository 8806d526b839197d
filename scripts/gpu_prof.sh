set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
KR='regex:diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel|unpack_dense'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" --csv --log-file gpurun_out/launches_c3_rcm.csv python bench.py --steps 1 --warmup 3 --applies 5 --no-cpu-baseline --single-ordering > /dev/null 2> gpurun_out/ncu_launch.log
timeout 1500 ncu --set full --clock-control none --import-source on -k 'regex:diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel' -c 5 -o gpurun_out/prof_c3_rcm python bench.py --steps 1 --warmup 3 --applies 3 --no-cpu-baseline --single-ordering > /dev/null 2> gpurun_out/ncu_full.log
tail -2 gpurun_out/ncu_full.log
