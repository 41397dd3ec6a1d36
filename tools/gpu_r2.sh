set -x
timeout 300 python tools/summarize_probe.py > gpurun_out/r2_summ.log 2>&1; tail -6 gpurun_out/r2_summ.log
SSB_BUILD_TRACE=1 timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 > gpurun_out/r2_build10m.log 2>&1; tail -40 gpurun_out/r2_build10m.log
timeout 600 python tools/build_profile.py --rows 25000000 --tau 100000 > gpurun_out/r2_build25m.log 2>&1; tail -3 gpurun_out/r2_build25m.log
