# Thin (P Q)^T-row tasks load only the live 128-byte pieces of A: full GPU suite, timings, c3 bench line.
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/thin_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/thin_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/thin_smoke.log 2>&1; echo "smoke exit $?"
for c in c3 c4 c5; do timeout 600 python scripts/factor_bench.py $c 5; done
timeout 900 python bench.py > gpurun_out/thin_bench_c3.json 2> gpurun_out/thin_bench_c3.err; echo "bench exit $?"
