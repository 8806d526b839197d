# Level-scheduled factorization launches (+ fused group assembly): parity + timings.
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_factor.py -x -q -p no:cacheprovider > gpurun_out/levels_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/levels_pytest.log
for c in c3 c4 c5 c2; do
  timeout 600 python scripts/factor_bench.py $c 5
  FETI_SP_LEVELS=0 timeout 600 python scripts/factor_bench.py $c 5
done
FETI_SP_GROUPS=4 timeout 600 python scripts/factor_bench.py c3 5
FETI_SP_GROUPS=16 timeout 600 python scripts/factor_bench.py c3 5
