# Group assembly fused into the factorization graph: parity + timings.
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py -x -q -p no:cacheprovider > gpurun_out/fuse_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/fuse_pytest.log
for c in c3 c4 c5; do
  timeout 600 python scripts/factor_bench.py $c 5
  FETI_SP_FUSE=0 timeout 600 python scripts/factor_bench.py $c 5
  FETI_SP_PRIO=1 timeout 600 python scripts/factor_bench.py $c 5
done
