# Work-balanced (LPT) factorization groups: parity + timings.
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_pcpg.py -x -q -p no:cacheprovider > gpurun_out/lpt_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/lpt_pytest.log
for c in c3 c4 c5; do
  timeout 600 python scripts/factor_bench.py $c 5
  FETI_SP_ASSIGN=contiguous timeout 600 python scripts/factor_bench.py $c 5
done
timeout 900 python bench.py --no-cpu-baseline --no-solve > gpurun_out/lpt_bench_c3.json 2> gpurun_out/lpt_bench_c3.err; echo "bench c3 exit $?"
