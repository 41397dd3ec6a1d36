for w in 8 16 32; do echo "== warm $w"; SSB_TC_WARM=$w timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0,0.1 --ks 100 2>&1 | tail -2 | python -c "
import sys,json
for l in sys.stdin: j=json.loads(l); print('  ', j['sigma'], j['k'], j['ms'], j['cand_series'], {k:v[0] for k,v in j['kernels'].items()})"; done
for w in 4 8 16; do SSB_TC_WARM=$w timeout 900 python bench.py --workload c4 --steps 3 --warmup 2 --cpu-sample 0 > gpurun_out/b_c4w.json 2>/dev/null; python -c "
import json; j=json.load(open('gpurun_out/b_c4w.json')); print('c4 warm $w', j['value'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"; done
