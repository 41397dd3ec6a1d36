timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r12_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/r12_tests.log
timeout 300 python tools/summarize_probe.py 2>&1 | tail -4
timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 --repeat 2 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r12_c2.json 2>gpurun_out/r12_c2.err; echo "bench exit $?"; python -c "import json; j=json.load(open('gpurun_out/r12_c2.json')); print(j['value'], j['e2e'], j['build'])"
