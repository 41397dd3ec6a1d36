timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for w in c2 c1 c3 c4 c5; do
  timeout 1500 python bench.py --workload $w > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
  python -c "
import json; j=json.load(open('gpurun_out/b_$w.json')); print('$w', j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['frac'], j['build']['series_per_s'], j['cpu_baseline'] and round(j['cpu_baseline']['value'],2), j['clocks'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"
done
