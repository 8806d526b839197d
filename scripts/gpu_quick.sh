set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -3 gpurun_out/bench.log
