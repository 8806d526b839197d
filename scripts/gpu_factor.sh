set -x
timeout 900 python -m pytest tests/test_gpu_factor.py -x -q 2>&1 | tail -3
python bench.py --steps 3 --warmup 3 --single-ordering --no-cpu-baseline --no-solve > gpurun_out/bench_fac.json 2> gpurun_out/bench_fac.log
