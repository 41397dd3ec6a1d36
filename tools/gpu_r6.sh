timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r6_tests.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/r6_tests.log
for w in 16 32 0; do SSB_BSTATS_W=$w timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 2>&1 | tail -1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r6_build_launches.csv python tools/build_profile.py --rows 10000000 --tau 10000 --no-warm > gpurun_out/r6_ncu.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py launches gpurun_out/r6_build_launches.csv > gpurun_out/r6_launches.txt; head -12 gpurun_out/r6_launches.txt
