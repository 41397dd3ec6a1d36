for w in 16 32; do echo "W=$w"; SSB_STATS_W=$w timeout 300 python tools/summarize_probe.py 2>&1 | tail -4; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:build_eval_warp -s 10 -c 1 -o gpurun_out/r11_eval python tools/build_profile.py --rows 10000000 --tau 10000 --no-warm > gpurun_out/r11_ncu1.log 2>&1; echo "ncu1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:finalize_rows -c 1 -o gpurun_out/r11_fin python tools/build_profile.py --rows 10000000 --tau 10000 --no-warm > gpurun_out/r11_ncu2.log 2>&1; echo "ncu2 exit $?"
