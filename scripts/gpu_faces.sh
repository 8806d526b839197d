# Face-grown dissection ordering: parity of the sparse route + factorization timings c3/c4/c5.
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_headline.py -x -q -p no:cacheprovider > gpurun_out/faces_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/faces_pytest.log
for c in c3 c4 c5; do timeout 600 python scripts/factor_bench.py $c 5; done
for c in c3 c4; do FETI_SPARSE_ORDERING=dissection:2 timeout 600 python scripts/factor_bench.py $c 5; done
