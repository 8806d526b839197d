set -x
timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -3
timeout 1200 ncu --set full --clock-control none --import-source on -k 'regex:sp_potrf|sp_gemm' -s 300 -c 4 -o gpurun_out/prof_c5 python bench.py --config c5 --steps 1 --warmup 3 --applies 3 --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_c5_full.log
tail -3 gpurun_out/ncu_c5_full.log
