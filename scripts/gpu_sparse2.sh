set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_factor.py -x -q 2>&1 | tail -5
python bench.py --config c5 --steps 3 --warmup 3 --applies 100 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log
tail -3 gpurun_out/bench_c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_' --csv --log-file gpurun_out/launches_c5.csv python bench.py --config c5 --steps 1 --warmup 3 --applies 3 --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_c5_launch.log
