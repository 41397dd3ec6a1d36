# A/B of builds on the same box: SSB_LIB_VARIANT selects libseriesearch_b200.<variant>.so
for v in head side; do
  export SSB_LIB_VARIANT=$v
  timeout 900 python bench.py --workload c4 --steps 3 --warmup 2 --cpu-sample 0 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json; j=json.load(open('gpurun_out/ab_$v.json')); print('$v', j['value'], j['ms_per_step'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"
done
