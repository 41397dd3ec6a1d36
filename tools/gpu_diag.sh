for w in c4 c5; do
  timeout 1500 python bench.py --workload $w --steps 3 --warmup 2 --cpu-sample 1 > gpurun_out/b_$w.json 2> gpurun_out/b_$w.err
  python -c "
import json; j=json.load(open('gpurun_out/b_$w.json')); print('$w', j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['frac'], j['build'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"
done
