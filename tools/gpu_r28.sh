# r28: C4 (k=100) K-tc epilogue share: full vs pipeline-only (diag 1) vs TMEM loads + max (diag 2)
for d in 0 1 2; do SSB_TC_DIAG=$d timeout 900 python bench.py --workload c4 --no-cpu-baseline --ingest-gb 0 --steps 5 > gpurun_out/r28_c4_$d.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r28_c4_$d.json')); print('c4 diag $d', j['value'], j['roofline']['avg_launch_ms'], j['kernels'], j['clocks'])"; done
SSB_TC_TRACE=1 timeout 900 python bench.py --workload c4 --no-cpu-baseline --ingest-gb 0 --steps 1 --warmup 0 2>&1 >/dev/null | grep "tc batch" | tail -3
