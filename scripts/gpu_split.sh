# Split forward-solve chains in the sparse route's group assembly: parity + timings.
set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q -p no:cacheprovider > gpurun_out/split_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/split_pytest.log
for c in c3 c4; do
  for s in 0 4 6 8; do FETI_TRSM_SEG=$s timeout 600 python scripts/factor_bench.py $c 5; done
done
FETI_TRSM_SEG=6 FETI_SP_GROUPS=12 timeout 600 python scripts/factor_bench.py c3 5
FETI_TRSM_SEG=6 FETI_SP_GROUPS=16 timeout 600 python scripts/factor_bench.py c3 5
FETI_TRSM_SEG=0 timeout 600 python scripts/factor_bench.py c5 5
FETI_TRSM_SEG=6 timeout 600 python scripts/factor_bench.py c5 5
