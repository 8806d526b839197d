timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_factor.py -x -q 2>&1 | tail -2
timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 20 > gpurun_out/b_c3s.json 2>/dev/null
timeout 400 python bench.py --config c5 --steps 3 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c5s.json 2>/dev/null
python -c "
import json
for f in ('b_c3s','b_c5s'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['value'], d['phases_ms'], d['e2e']['value'], d['roofline']['frac'])
"
