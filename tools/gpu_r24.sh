# r24: 32-column K-chunks (SWIZZLE_64B) for n = 96: tests, then C3 A/B against 64-column chunks
timeout 900 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -3
for cw in 64 32 64 32; do for d in 0 1 3 4; do SSB_TC_CW=$cw SSB_TC_DIAG=$d timeout 600 python bench.py --workload c3 --no-cpu-baseline --steps 10 > gpurun_out/r24_c3_$cw$d.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r24_c3_$cw$d.json')); print('c3 cw $cw diag $d', j['value'], j['roofline']['avg_launch_ms'], j['roofline']['frac'])"; done; done
