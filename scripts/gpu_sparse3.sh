set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -3
for G in 4 2; do
FETI_SP_GROUPS=$G python bench.py --config c5 --steps 3 --warmup 3 --applies 50 --no-cpu-baseline > gpurun_out/bench_c5_g$G.json 2> gpurun_out/bench_c5_g$G.log
done
