timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
for v in head new; do
  export SSB_LIB_VARIANT=$v
  echo "== $v"; timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0 --ks 1,10 2>&1 | tail -2 | python -c "
import sys,json
for l in sys.stdin: j=json.loads(l); print(j['k'], j['ms'], j['cand_series'], {k:v[0] for k,v in j['kernels'].items()})"
done
unset SSB_LIB_VARIANT
timeout 300 python bench.py --per-cell --cpu-sample 0 > gpurun_out/b_c2_cell.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/b_c2_cell.json')); print('per-cell', j['value'], j['e2e']['value'], j['ms_per_step'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"
timeout 300 python bench.py > gpurun_out/b_c2.json 2>&1; python -c "
import json; j=json.load(open('gpurun_out/b_c2.json')); print('by-k', j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['frac'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"
