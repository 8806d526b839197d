# Per-group step graphs (init on the group stream, per-group K readiness): parity + timings (value and e2e).
set -x
timeout 1500 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_pcpg.py tests/test_gpu_factor.py -x -q -p no:cacheprovider > gpurun_out/grpgraph_pytest.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/grpgraph_pytest.log
for c in c3 c4 c5; do timeout 600 python scripts/factor_bench.py $c 5; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/grpgraph_bench_c3.json 2> gpurun_out/grpgraph_bench_c3.err; echo "bench c3 exit $?"
timeout 1200 python bench.py --config c5 --no-cpu-baseline --no-solve > gpurun_out/grpgraph_bench_c5.json 2> gpurun_out/grpgraph_bench_c5.err; echo "bench c5 exit $?"
