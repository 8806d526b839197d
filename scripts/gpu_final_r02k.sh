# Final-code evidence, part 2: 2-rank time-shared bench through the fused exchange, reference arm, c1/c2 lines.
set -x
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --sparse-only --no-cpu-baseline --no-solve --steps 3 --warmup 3 \
  > gpurun_out/r02k_bench_c3_2rank_gloo_1gpu.json 2> gpurun_out/r02k_bench_2rank.err; echo "2rank exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02k_bench_c3_reference_arm.json \
  2> gpurun_out/r02k_bench_ref.err; echo "ref exit $?"
timeout 600 python bench.py --config c2 --route sparse > gpurun_out/r02k_bench_c2_sparse.json 2> gpurun_out/r02k_bench_c2.err; echo "c2 exit $?"
timeout 600 python bench.py --config c1 --route sparse > gpurun_out/r02k_bench_c1_sparse.json 2> gpurun_out/r02k_bench_c1.err; echo "c1 exit $?"
