#!/bin/bash
# The round's committed measurements (GPU box): bench lines per config, the
# reference arm, the ncu launch list of the default bench, --set full captures
# of the dominant kernels, the single-query probes.  Outputs under gpurun_out/;
# the summaries worth keeping are copied to profiles/ by hand (tools/ncu_summary.py).
#   bash tools/profile_round.sh r02 [parts]   parts: bench ref launches full probes (default: all)
set -u
TAG=${1:-r02}
PARTS=${2:-"bench ref launches full probes"}
O=gpurun_out
make -s -j8 -C paper_2212_13297_b200/csrc
for p in $PARTS; do
case $p in
bench)
  timeout 900 python bench.py > $O/${TAG}_bench_c4.json 2> $O/${TAG}_bench_c4.err; tail -3 $O/${TAG}_bench_c4.err
  for w in c1 c2 c3 c5; do
    timeout 1200 python bench.py --workload $w > $O/${TAG}_bench_$w.json 2> $O/${TAG}_bench_$w.err; tail -2 $O/${TAG}_bench_$w.err
  done ;;
ref)
  timeout 900 python bench.py --impl reference > $O/${TAG}_bench_reference_c4.json 2> $O/${TAG}_bench_reference_c4.err ;;
launches)
  # the query step's kernels (the two timed builds launch ~800 kernels first: filter by name)
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"tc_filter|rescore|ix_|select|proj_b|proj_t|proj_m|proj_q|query_prep|keys_to|seed_bound|merge|pack" -c 600 --csv \
    --log-file $O/${TAG}_c4_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --ingest-gb 0 \
    > $O/${TAG}_c4_launches.log 2>&1 ;;
full)
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:tc_filter -s 3 -c 1 \
    -o $O/${TAG}_c4_tc python bench.py --steps 1 --warmup 1 --no-cpu-baseline --ingest-gb 0 > $O/${TAG}_ncu_c4.log 2>&1
  timeout 1500 ncu --set full --import-source on --clock-control none -k regex:tc_filter -s 12 -c 1 \
    -o $O/${TAG}_c3_tc python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline --ingest-gb 0 > $O/${TAG}_ncu_c3.log 2>&1
  timeout 1500 ncu --set full --clock-control none -k regex:"words_kernel|segment_stats" -c 4 \
    -o $O/${TAG}_summarize python tools/summarize_probe.py > $O/${TAG}_ncu_summarize.log 2>&1
  timeout 1500 ncu --set full --clock-control none -k regex:"ix_|scan_rows" -s 40 -c 12 \
    -o $O/${TAG}_ix python tools/latency_probe.py --workload c2 --queries 200 --single 4 --routes tree \
    > $O/${TAG}_ncu_ix.log 2>&1 ;;
probes)
  timeout 900 python tools/latency_probe.py --workload c2 --queries 1000 --single 30 --routes tree,tensor,auto \
    > $O/${TAG}_lat_c2.jsonl 2> $O/${TAG}_lat_c2.err
  timeout 1200 python tools/latency_probe.py --workload c4 --queries 200 --single 20 --routes auto,tensor \
    > $O/${TAG}_lat_c4.jsonl 2> $O/${TAG}_lat_c4.err ;;
esac
done
