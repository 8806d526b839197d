timeout 300 python -m pytest tests/test_gpu_sparse.py -x -q -k "matches_reference or bit_repro or spd" tests/test_gpu_factor.py 2>&1 | tail -1
timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 50 > gpurun_out/b_c3s.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/b_c3s.json')); print(d['value'], d['phases_ms']['ms_factorize'], d['e2e']['value'], d['host_side_ms'], d['apply']['e2e_ms_per_iter'])
"
