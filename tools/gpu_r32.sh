# r32: C2 k=10 epilogue knobs: buckets off, refresh period
run() { env $1 timeout 600 python bench.py --no-cpu-baseline --ingest-gb 0 --steps 20 --per-cell > gpurun_out/r32_$2.json 2>/dev/null; python -c "import json; j=json.load(open('gpurun_out/r32_$2.json')); print('$2', j['value'], j['roofline']['avg_launch_ms'], j['kernels']['tc_filter']['launches'], j['kernels']['rescore']['ms'])"; }
for i in 1 2; do run X=1 base; run SSB_TC_NOBUCKET=1 nobucket; run SSB_TC_RMASK=15 r15; run SSB_TC_RMASK=3 r3; done
