SSB_BUILD_TRACE=1 timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 --repeat 2 > gpurun_out/r9_trace.log 2>&1; grep -v "stats buffer" gpurun_out/r9_trace.log | tail -60
