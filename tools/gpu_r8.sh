timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r8_tests.log 2>&1; echo "tests exit $?"; tail -3 gpurun_out/r8_tests.log
timeout 600 python tools/build_profile.py --rows 10000000 --tau 10000 --repeat 2 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r8_build_launches.csv python tools/build_profile.py --rows 10000000 --tau 10000 --no-warm > gpurun_out/r8_ncu.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py launches gpurun_out/r8_build_launches.csv > gpurun_out/r8_launches.txt; head -8 gpurun_out/r8_launches.txt
