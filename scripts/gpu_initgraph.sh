# Pool init + K scatter per group inside the step graph; ordering cache: parity + timings.
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_headline.py tests/test_gpu_pcpg.py -x -q -p no:cacheprovider > gpurun_out/initgraph_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/initgraph_pytest.log
for c in c3 c4 c5; do
  timeout 600 python scripts/factor_bench.py $c 5
  FETI_SP_INIT_GRAPH=0 timeout 600 python scripts/factor_bench.py $c 5
done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/initgraph_bench_c3.json 2> gpurun_out/initgraph_bench_c3.err; echo "bench exit $?"
FETI_SP_INIT_GRAPH=0 timeout 900 python bench.py --no-cpu-baseline --sparse-only --no-solve > gpurun_out/initgraph0_bench_c3.json 2> gpurun_out/initgraph0_bench_c3.err; echo "bench0 exit $?"
