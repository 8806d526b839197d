# Round-2 final evidence (face ordering, per-group step graphs, LPT groups): full GPU suite, smoke,
# bench lines c3 (default) / c4 / c5 / c2, 2-rank time-shared bench, reference arm, c3 step launch list.
set -x
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02i_pytest_gpu.log 2>&1
echo "pytest exit $?"; tail -3 gpurun_out/r02i_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r02i_bench_c3.json 2> gpurun_out/r02i_bench_c3.err; echo "c3 exit $?"
timeout 900 python bench.py --config c4 > gpurun_out/r02i_bench_c4.json 2> gpurun_out/r02i_bench_c4.err; echo "c4 exit $?"
timeout 1200 python bench.py --config c5 > gpurun_out/r02i_bench_c5.json 2> gpurun_out/r02i_bench_c5.err; echo "c5 exit $?"
timeout 600 python bench.py --config c2 --route sparse > gpurun_out/r02i_bench_c2_sparse.json 2> gpurun_out/r02i_bench_c2.err; echo "c2 exit $?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --dist-backend gloo --sparse-only --no-cpu-baseline --no-solve --steps 3 --warmup 3 \
  > gpurun_out/r02i_bench_c3_2rank_gloo_1gpu.json 2> gpurun_out/r02i_bench_2rank.err; echo "2rank exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02i_bench_c3_reference_arm.json \
  2> gpurun_out/r02i_bench_ref.err; echo "ref exit $?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k 'regex:sp_|diag_inverse|block_scale|trsm_chain|syrk_kernel' --csv \
  --log-file gpurun_out/r02i_c3_launches.csv python scripts/factor_bench.py c3 1 > gpurun_out/r02i_ncu1.log 2>&1
echo "ncu exit $?"
