# potrf stride 132: factor/sparse GPU parity subset, c3/c4 sparse-route bench
set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --sparse-only --no-cpu-baseline > gpurun_out/stride_c3.json 2> gpurun_out/stride_c3.log
python bench.py --config c4 --steps 3 --warmup 3 --sparse-only --no-cpu-baseline > gpurun_out/stride_c4.json 2> gpurun_out/stride_c4.log
python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/stride_c5.json 2> gpurun_out/stride_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel' --csv --log-file gpurun_out/launches_stride.csv python bench.py --steps 1 --warmup 3 --applies 5 --sparse-only --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launch_stride.log
