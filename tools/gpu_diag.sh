timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_index.py -q -x 2>&1 | tail -1
for o in leaf hash leaf hash; do echo "== $o"; SSB_TC_ROWORDER=$o timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0,0.01 --ks 1,10 2>&1 | tail -4 | python -c "
import sys,json
for l in sys.stdin: j=json.loads(l); print(j['sigma'], j['k'], j['ms'], j['cand_series'], {k:v[0] for k,v in j['kernels'].items()})"; done
