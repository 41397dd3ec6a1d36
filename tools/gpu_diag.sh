timeout 600 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
timeout 900 python bench.py --workload c3 > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
python -c "
import json; j=json.load(open('gpurun_out/b_c3.json')); print('c3', j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['frac'], {k:(round(v['ms'],1),v['launches']) for k,v in j['kernels'].items()})"
