SSB_TC_TRACE=1 timeout 900 python bench.py --workload c4 --route tensor --steps 1 --warmup 1 --cpu-sample 0 > gpurun_out/b_c4_tensor.json 2> gpurun_out/b_c4_tensor.err
grep ssb gpurun_out/b_c4_tensor.err | head
SSB_TC_TRACE=1 timeout 900 python bench.py --workload c2 --steps 1 --warmup 1 --cpu-sample 0 2>&1 >/dev/null | grep ssb | head -20
