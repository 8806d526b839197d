timeout 900 python -m pytest tests/test_gpu_sparse.py -x -q -k "matches_reference or c3" 2>&1 | tail -1
for F in prio flat; do
if [ $F = flat ]; then export FETI_SP_FLAT=1; fi
timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 20 > gpurun_out/b_c3_$F.json 2>/dev/null
timeout 400 python bench.py --config c5 --steps 3 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c5_$F.json 2>/dev/null
done
python -c "
import json
for f in ('b_c3_prio','b_c3_flat','b_c5_prio','b_c5_flat'):
    d=json.load(open('gpurun_out/'+f+'.json')); p=d['phases_ms']; print(f, d['value'], p['ms_factorize'], p['ms_assembly_tail'], d['e2e']['value'])
"
