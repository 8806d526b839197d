# apply kernel: warp count / register buffer depth A/B (GPU parity subset + c3/c4 sparse-route bench)
set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "apply or golden" 2>&1 | tail -3
for v in 3buf 2buf; do
  if [ $v = 2buf ]; then export FETI_APPLY_2BUF=1; fi
  python bench.py --config c4 --steps 3 --warmup 3 --sparse-only --no-cpu-baseline > gpurun_out/bench_c4_$v.json 2> gpurun_out/bench_c4_$v.log
  python bench.py --steps 3 --warmup 3 --sparse-only --no-cpu-baseline > gpurun_out/bench_c3_$v.json 2> gpurun_out/bench_c3_$v.log
done
python - <<'PY'
import json
for f in ("bench_c4_3buf", "bench_c4_2buf", "bench_c3_3buf", "bench_c3_2buf"):
    d = json.loads(open(f"gpurun_out/{f}.json").read().strip().splitlines()[-1])
    print(f, d["value"], d["e2e"]["value"], d["apply"]["kernel_ms_per_iter"], d["apply"]["roofline"]["frac"])
PY
