# r34: staged contiguous-segment statistics output: parity + A/B
timeout 900 python -m pytest tests/test_gpu_scan.py tests/test_gpu_index.py -q -x 2>&1 | tail -2
for v in head new head new; do
  export SSB_LIB_VARIANT=$v
  echo "== $v"; timeout 300 python tools/summarize_probe.py 2>&1 | grep segment_stats
done
