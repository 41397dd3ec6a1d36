# r26: device generator tests + C2/C3 bench with build.device_gen
timeout 900 python -m pytest tests/test_gpu_generate.py -q -x 2>&1 | tail -3
for w in c2 c3; do timeout 600 python bench.py --workload $w --no-cpu-baseline --steps 10 > gpurun_out/r26_$w.json 2> gpurun_out/r26_$w.err; echo "bench $w exit $?"; python -c "import json; j=json.load(open('gpurun_out/r26_$w.json')); print(j['value'], j['build'].get('device_gen'), j['build'].get('ingest',{}).get('GBps'))"; done
