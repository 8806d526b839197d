# Re-entry check of HEAD on a fresh B200: full -m gpu suite, smoke, default bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02f_pytest_gpu.log 2>&1
echo "pytest exit $?"
tail -5 gpurun_out/r02f_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1
echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
echo "bench exit $?"
cat gpurun_out/r02f_bench.json | head -c 3000
