# r36: final state: smoke, full GPU tests, C1-C5 bench lines, C2 launch list
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for w in c2 c1 c3 c4 c5; do timeout 1200 python bench.py --workload $w > gpurun_out/r36_bench_$w.json 2> gpurun_out/r36_bench_$w.err; echo "$w exit $?"; python -c "import json; j=json.load(open('gpurun_out/r36_bench_$w.json')); print('$w', j['value'], j['e2e']['value'], j['roofline']['frac'], j['build']['series_per_s'], j['build'].get('roofline',{}).get('frac'), j['clocks'])"; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r36_c2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --ingest-gb 0 > gpurun_out/r36_ncu_launch.log 2>&1; echo "ncu launches exit $?"
