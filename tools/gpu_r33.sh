# r33: float64 division by segment widths via the reciprocal table (Markstein): parity + A/B
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for v in head new head new; do
  export SSB_LIB_VARIANT=$v
  echo "== $v"; timeout 300 python tools/summarize_probe.py 2>&1 | grep segment_stats
  timeout 300 python tools/build_profile.py --rows 10000000 2>&1 | tail -1 | cut -c1-240
done
