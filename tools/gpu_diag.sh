for cs in 2 4 1; do for d in 1 0; do echo "cs=$cs diag=$d"; SSB_TC_CSMAX=$cs SSB_TC_DIAG=$d timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0 --ks 1,10 2>&1 | tail -2 | python -c "
import sys,json
for l in sys.stdin: j=json.loads(l); print('  ', j['k'], j['ms'], j['cand_series'], {k:v[0] for k,v in j['kernels'].items()})"; done; done
