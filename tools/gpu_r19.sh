# r19: health check of the restored tree on a fresh box + C3 K-tc diagnosis
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r19_smoke.log 2>&1; echo "smoke exit $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r19_pytest.log 2>&1; echo "pytest exit $?"; tail -3 gpurun_out/r19_pytest.log
timeout 600 python bench.py > gpurun_out/r19_bench_c2.json 2> gpurun_out/r19_bench_c2.err; echo "bench exit $?"; cut -c1-400 gpurun_out/r19_bench_c2.json
for d in 0 1 2; do SSB_TC_DIAG=$d timeout 600 python bench.py --workload c3 --no-cpu-baseline --steps 5 > gpurun_out/r19_c3_diag$d.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r19_c3_diag$d.json')); print('c3 diag $d', j['value'], j['roofline']['avg_launch_ms'], j['kernels'])"; done
SSB_TC_TRACE=1 timeout 600 python bench.py --workload c3 --no-cpu-baseline --steps 1 --warmup 0 > /dev/null 2> gpurun_out/r19_c3_trace.err; tail -20 gpurun_out/r19_c3_trace.err
