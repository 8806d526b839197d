for G in 2 4 8; do
FETI_SP_GROUPS=$G timeout 300 python bench.py --config c3 --sparse-only --steps 5 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c3_g$G.json 2>/dev/null
FETI_SP_GROUPS=$G timeout 400 python bench.py --config c5 --steps 3 --warmup 3 --applies 20 --no-cpu-baseline > gpurun_out/b_c5_g$G.json 2>/dev/null
done
python -c "
import json
for G in (2,4,8):
  for c in ('c3','c5'):
    d=json.load(open(f'gpurun_out/b_{c}_g{G}.json')); p=d['phases_ms']; print(c, G, d['value'], p['ms_factorize'], p['ms_assembly_tail'], d['e2e']['value'])
"
