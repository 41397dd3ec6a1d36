timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_index.py -q -x 2>&1 | tail -2
for d in 0 1; do
  echo "diag=$d"
  SSB_TC_DIAG=$d timeout 120 python tools/cell_profile.py --rows 1000000 --sigmas 1.0,0.01 --ks 1,10 2>&1 | tail -4 | cut -c1-300
done
