timeout 300 python -m pytest tests/test_gpu_sparse.py -x -q -k "matches_reference or bit_repro or spd" 2>&1 | tail -3
timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 50 > gpurun_out/b_c3_dag.json 2>/dev/null
FETI_SP_DAG=0 timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 50 > gpurun_out/b_c3_nodag.json 2>/dev/null
timeout 400 python bench.py --config c5 --steps 3 --warmup 3 --applies 50 --no-cpu-baseline > gpurun_out/b_c5_dag.json 2>/dev/null
python -c "
import json
for f in ('b_c3_dag','b_c3_nodag','b_c5_dag'):
    try:
        d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['value'], d['phases_ms']['ms_factorize'], d['e2e']['value'], d['roofline']['frac'])
    except Exception as e: print(f, 'failed', e)
"
