set -x
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
python bench.py --config c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.log
python bench.py --config c4 --steps 3 --warmup 3 --sparse-only --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel' --csv --log-file gpurun_out/launches_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 5 --sparse-only --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch.log
ls gpurun_out
