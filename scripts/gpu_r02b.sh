python scripts/factor_bench.py c3
python scripts/factor_bench.py c4 3
python scripts/apply_bench.py c3; python scripts/apply_bench.py c4
python scripts/apply_bench.py c2; FETI_APPLY_CPS=1 python scripts/apply_bench.py c2
python scripts/pcpg_bench.py c3 | tail -1
python -m pytest tests -q -x -p no:cacheprovider -m "gpu and not slow" 2>&1 | tail -2
python bench.py --config c2 --no-device-factor > gpurun_out/bench_c2b.json 2> gpurun_out/bench_c2b.err
