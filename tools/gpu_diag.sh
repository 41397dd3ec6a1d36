timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_tc.py -q -x 2>&1 | grep -v "Warning\|popen\|self.pid\|^$" | tail -25
timeout 600 python tools/build_profile.py --rows 10000000 2>&1 | tail -1
