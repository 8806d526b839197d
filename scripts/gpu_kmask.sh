# k-slice skipping in the sparse factorization's tile products: exactness + timings.
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_headline.py -x -q -p no:cacheprovider > gpurun_out/kmask_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/kmask_pytest.log
for c in c3 c4 c5; do
  timeout 600 python scripts/factor_bench.py $c 5
  FETI_SP_KMASK=0 timeout 600 python scripts/factor_bench.py $c 5
done
timeout 900 python bench.py --no-cpu-baseline --no-solve --sparse-only > gpurun_out/kmask_bench_c3.json 2> gpurun_out/kmask_bench_c3.err; echo "bench exit $?"
