timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r16_tests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/r16_tests.log
timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 --repeat 2 2>&1 | tail -1
timeout 600 python tools/build_profile.py --rows 25000000 --tau 100000 --repeat 2 2>&1 | tail -1
