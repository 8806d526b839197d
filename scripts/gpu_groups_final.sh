# Group count with per-group graphs + k-slice skipping: device (factor_bench) and e2e (bench) at c3 / c5.
set -x
for G in 8 12 16; do
  FETI_SP_GROUPS=$G timeout 600 python scripts/factor_bench.py c3 5
  FETI_SP_GROUPS=$G timeout 600 python scripts/factor_bench.py c5 5
done
for G in 8 16; do
  FETI_SP_GROUPS=$G timeout 900 python bench.py --no-cpu-baseline --no-solve --sparse-only > gpurun_out/groups${G}_bench_c3.json 2>/dev/null
  FETI_SP_GROUPS=$G timeout 900 python bench.py --config c5 --no-cpu-baseline --no-solve > gpurun_out/groups${G}_bench_c5.json 2>/dev/null
done
