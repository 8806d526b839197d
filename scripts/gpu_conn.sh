# Hardware work queues: CUDA_DEVICE_MAX_CONNECTIONS (default 8) vs the 8-16 group streams + context + copy streams.
set -x
for C in 8 16 32; do
  for G in 8 16; do
    CUDA_DEVICE_MAX_CONNECTIONS=$C FETI_SP_GROUPS=$G timeout 600 python scripts/factor_bench.py c3 5
  done
  CUDA_DEVICE_MAX_CONNECTIONS=$C timeout 600 python scripts/factor_bench.py c5 5
done
CUDA_DEVICE_MAX_CONNECTIONS=32 timeout 900 python bench.py --no-cpu-baseline --no-solve --sparse-only > gpurun_out/conn32_bench_c3.json 2>/dev/null
