# r35: ssb_query_multi: parity + C2 A/B (multi vs one call per k)
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
for m in "" "--no-multi"; do timeout 600 python bench.py --no-cpu-baseline --ingest-gb 0 $m > gpurun_out/r35_c2$m.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r35_c2$m.json')); print('c2 $m', j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['avg_launch_ms'], j['clocks']['sm_mhz'])"; done; done
