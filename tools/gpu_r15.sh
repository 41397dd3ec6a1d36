timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r15_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/r15_tests.log
timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 --repeat 2 2>&1 | tail -1
SSB_BUILD_TRACE=1 timeout 600 python tools/build_profile.py --rows 10000000 --n 96 --tau 10000 --repeat 2 > gpurun_out/r15_trace96.log 2>&1; tail -40 gpurun_out/r15_trace96.log
