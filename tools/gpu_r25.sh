# r25: ingest pipeline tests + build_index from file + C2 bench with build.ingest
timeout 900 python -m pytest tests/test_gpu_ingest.py tests/test_gpu_index.py -q -x 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/r25_c2.json 2> gpurun_out/r25_c2.err; echo "bench exit $?"; python -c "import json; j=json.load(open('gpurun_out/r25_c2.json')); print(j['value'], j['build'].get('ingest'))"
