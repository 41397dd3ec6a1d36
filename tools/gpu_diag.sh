timeout 300 python -m pytest tests/test_gpu_tc.py tests/test_gpu_index.py -q -x 2>&1 | tail -1
timeout 60 python tools/cell_profile.py --rows 1000000 --sigmas 1.0 --ks 1,10 2>&1 | tail -2 | cut -c1-300
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; head -c 700 gpurun_out/b_c2.json
