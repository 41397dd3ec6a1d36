set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1_gpu_tests.log 2>&1; echo "tests exit $?"
tail -3 gpurun_out/r1_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/r1_bench_c2.json 2> gpurun_out/r1_bench_c2.err; echo "bench exit $?"
cat gpurun_out/r1_bench_c2.json | head -c 1500
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1_bench_ref.json 2>gpurun_out/r1_bench_ref.err; echo "ref exit $?"
cat gpurun_out/r1_bench_ref.json | head -c 800
