timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r14_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/r14_tests.log
timeout 300 python tools/summarize_probe.py 2>&1 | tail -4
timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 --repeat 2 2>&1 | tail -1
timeout 900 python bench.py --workload c3 > gpurun_out/r14_c3.json 2> gpurun_out/r14_c3.err; echo "c3 exit $?"; python -c "import json; j=json.load(open('gpurun_out/r14_c3.json')); print(j['value'], j['build'])"
