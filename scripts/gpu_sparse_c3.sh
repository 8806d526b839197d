set -x
for C in c3 c4 c2; do
python bench.py --config $C --route sparse --steps 3 --warmup 3 --applies 50 --no-cpu-baseline > gpurun_out/bench_${C}_sparse.json 2> gpurun_out/bench_${C}_sparse.log
tail -2 gpurun_out/bench_${C}_sparse.log
done
