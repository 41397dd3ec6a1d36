# r21: A/B TC_RS 4 (head) vs 8 (new) on C3 / C2
export SSB_LIB_VARIANT=new
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
for v in head new head new; do
  export SSB_LIB_VARIANT=$v
  for d in 0 1; do SSB_TC_DIAG=$d timeout 600 python bench.py --workload c3 --no-cpu-baseline --steps 10 > gpurun_out/r21_c3_$v$d.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r21_c3_$v$d.json')); print('c3 $v diag $d', j['value'], j['roofline']['avg_launch_ms'], j['roofline']['frac'])"; done
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r21_c2_$v.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r21_c2_$v.json')); print('c2 $v', j['value'], j['roofline']['avg_launch_ms'], j['roofline']['frac'])"
done
