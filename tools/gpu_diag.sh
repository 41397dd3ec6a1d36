timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
echo diag1; SSB_TC_DIAG=1 timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0 --ks 1 2>&1 | tail -1 | cut -c1-300
timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0 --ks 1,10 2>&1 | tail -2 | cut -c1-300
