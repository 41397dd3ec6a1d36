# r20: ncu of the C3 tc_filter (full epilogue and pipeline-only)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_filter -s 4 -c 1 -o gpurun_out/r20_c3_tc python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r20_ncu0.log 2>&1; echo "ncu c3 exit $?"
SSB_TC_DIAG=1 timeout 900 ncu --set full --clock-control none -k regex:tc_filter -s 4 -c 1 -o gpurun_out/r20_c3_tc_diag1 python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r20_ncu1.log 2>&1; echo "ncu c3 diag1 exit $?"
