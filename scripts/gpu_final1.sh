set -x
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --single-ordering --no-device-factor --no-solve --applies 20 > gpurun_out/bench_2rank_c3.json 2> gpurun_out/bench_2rank_c3.log
tail -3 gpurun_out/bench_2rank_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel|apply_kernel|reduce_kernel' --csv --log-file gpurun_out/launches_c3_sparse.csv python bench.py --steps 1 --warmup 3 --applies 5 --sparse-only > /dev/null 2> gpurun_out/ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:sp_gemm8|sp_potrf|apply_kernel|trsm_chain|syrk_kernel' -s 300 -c 8 -o gpurun_out/prof_c3_sparse python bench.py --steps 1 --warmup 3 --applies 3 --sparse-only > /dev/null 2> gpurun_out/ncu_full.log
ls gpurun_out
