# A/B of builds on the same box: SSB_LIB_VARIANT selects libseriesearch_b200.<variant>.so
export SSB_LIB_VARIANT=new
timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_index.py -q -x 2>&1 | tail -1
for v in head new head new; do
  export SSB_LIB_VARIANT=$v
  echo "== $v"; timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0 --ks 33,100 2>&1 | tail -2 | python -c "
import sys,json
for l in sys.stdin: j=json.loads(l); print(j['k'], j['ms'], j['cand_series'], {k:v[0] for k,v in j['kernels'].items()})"
done
