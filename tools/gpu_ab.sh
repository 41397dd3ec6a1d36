# A/B of builds on the same box: SSB_LIB_VARIANT selects libseriesearch_b200.<variant>.so
export SSB_LIB_VARIANT=new
timeout 600 python -m pytest tests/test_gpu_index.py -q -x 2>&1 | tail -1
for v in head new head new; do
  export SSB_LIB_VARIANT=$v
  echo "== $v"; timeout 300 python tools/build_profile.py --rows 10000000 2>&1 | tail -1 | cut -c1-200
done
