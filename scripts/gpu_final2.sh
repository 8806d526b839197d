set -x
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log
tail -2 gpurun_out/bench_ref.log
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:sp_gemm8|sp_potrf' --csv --log-file gpurun_out/traffic_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 3 --sparse-only --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_traffic.log
ls -la gpurun_out
