set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --dist-backend gloo --single-ordering --applies 20 > gpurun_out/bench_2rank_c2.json 2> gpurun_out/bench_2rank_c2.log
tail -3 gpurun_out/bench_2rank_c2.log
python bench.py --config c2 --steps 3 --warmup 3 --single-ordering --no-cpu-baseline --applies 50 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
tail -3 gpurun_out/bench_c4.log
