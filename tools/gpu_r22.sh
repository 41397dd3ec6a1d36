# r22: C3 cluster size 1 vs 2 (TC_RS 8 build)
for cs in 2 1 2 1; do
  for d in 0 1; do SSB_TC_CSMAX=$cs SSB_TC_DIAG=$d timeout 600 python bench.py --workload c3 --no-cpu-baseline --steps 10 > gpurun_out/r22_c3_$cs$d.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r22_c3_$cs$d.json')); print('c3 cs $cs diag $d', j['value'], j['roofline']['avg_launch_ms'], j['roofline']['frac'])"; done
done
