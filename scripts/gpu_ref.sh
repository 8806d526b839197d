set -x
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
tail -3 gpurun_out/bench_ref.log
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g | head -2
