# Last check of HEAD: full GPU suite, smoke, default bench.
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/head_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -2 gpurun_out/head_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/head_bench_c3.json 2> gpurun_out/head_bench_c3.err; echo "bench exit $?"
