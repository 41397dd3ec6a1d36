timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r3_build_launches.csv python tools/build_profile.py --rows 10000000 --tau 10000 --no-warm > gpurun_out/r3_ncu.log 2>&1; echo "ncu exit $?"
python tools/ncu_summary.py launches gpurun_out/r3_build_launches.csv | head -40
