# r27: no trailing sync in ssb_query: full GPU tests + C2 bench
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r27_c2_$i.json 2> gpurun_out/r27_c2.err; python -c "import json; j=json.load(open('gpurun_out/r27_c2_$i.json')); print(j['value'], j['e2e']['value'], j['ms_per_step'], j['roofline']['avg_launch_ms'], j['clocks'])"; done
