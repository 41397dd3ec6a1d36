timeout 900 python -m pytest tests/test_gpu_index.py -q -x 2>&1 | tail -1
timeout 600 python tools/build_profile.py --rows 10000000 2>&1 | tail -1
SSB_BUILD_TRACE=1 timeout 900 python tools/build_profile.py --rows 20000000 --tau 100000 2>&1 | grep -v "^\[ssb build\] level" | tail -6
