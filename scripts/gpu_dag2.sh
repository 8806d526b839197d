for V in 0 1; do
FETI_SP_DAG=$V timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c3_dag$V.json 2>/dev/null
FETI_SP_DAG=$V timeout 400 python bench.py --config c5 --steps 3 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c5_dag$V.json 2>/dev/null
done
python -c "
import json
for f in ('b_c3_dag0','b_c3_dag1','b_c5_dag0','b_c5_dag1'):
    d=json.load(open('gpurun_out/'+f+'.json')); p=d['phases_ms']; print(f, d['value'], p['ms_factorize'], p['ms_assembly_tail'])
"
