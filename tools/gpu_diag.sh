timeout 600 python -m pytest tests/test_gpu_tc.py tests/test_gpu_index.py -q -x 2>&1 | tail -1
for w in c1 c2; do
  timeout 900 python bench.py --workload $w > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
  python -c "
import json; j=json.load(open('gpurun_out/b_$w.json')); print('$w', j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['frac'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()}, j['gpu_launches'])"
done
