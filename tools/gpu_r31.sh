# r31: A/B per-thread (head) vs per-warp (new) TMEM release arrives: C3 and C2
export SSB_LIB_VARIANT=new
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_index.py -q -x 2>&1 | tail -1
for v in head new head new; do
  export SSB_LIB_VARIANT=$v
  for d in 0 1 4; do SSB_TC_DIAG=$d timeout 600 python bench.py --workload c3 --no-cpu-baseline --ingest-gb 0 --steps 10 > gpurun_out/r31_c3_$v$d.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r31_c3_$v$d.json')); print('c3 $v diag $d', j['value'], j['roofline']['avg_launch_ms'], j['roofline']['frac'])"; done
  timeout 600 python bench.py --no-cpu-baseline --ingest-gb 0 --steps 10 > gpurun_out/r31_c2_$v.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r31_c2_$v.json')); print('c2 $v', j['value'], j['roofline']['avg_launch_ms'], j['roofline']['frac'])"
done
