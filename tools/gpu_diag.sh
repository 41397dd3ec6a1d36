# r01 per-kernel ncu evidence (SpeedOfLight + DRAM bytes)
M="--section SpeedOfLight --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none"
timeout 900 ncu $M -k regex:"build_stats|build_eval|build_minmax|layout_rows|words_kernel|to_bf16|build_scatter|build_flags" -c 60 -o gpurun_out/k_build python tools/build_profile.py --rows 10000000 --no-warm > gpurun_out/k1.log 2>&1
timeout 900 ncu $M -k regex:"scan_dense|select_topk" -s 4 -c 4 -o gpurun_out/k_brute python bench.py --engine bruteforce --steps 1 --warmup 1 --cpu-sample 0 > gpurun_out/k3.log 2>&1
tail -n 1 gpurun_out/k1.log; tail -n 1 gpurun_out/k3.log
