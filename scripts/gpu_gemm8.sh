timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -1
for V in 8 9; do
if [ $V = 9 ]; then export FETI_SP_GEMM9=1; fi
timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 20 > gpurun_out/b_c3_$V.json 2>/dev/null
timeout 400 python bench.py --config c5 --steps 3 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c5_$V.json 2>/dev/null
done
python -c "
import json
for f in ('b_c3_8','b_c3_9','b_c5_8','b_c5_9'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, d['value'], d['phases_ms']['ms_factorize'], d['e2e']['value'], d['roofline']['frac'])
"
