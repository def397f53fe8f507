O=gpurun_out/s4r; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lane_lists or c2_whole or overlapped or composite or render_records or session_matches" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
for ll in 0 1; do
  AB_TAG="lanes$ll 5-64" VMSPLAT_LANE_LISTS=$ll timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="lanes$ll 5-34" AB_TO=35 VMSPLAT_LANE_LISTS=$ll timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
for mg in 0 4; do
  AB_TAG="lanes1 margin$mg 5-34" AB_TO=35 VMSPLAT_LANE_MARGIN=$mg timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
AB_TAG="lanes2 5-34" AB_TO=35 VMSPLAT_LANE_LISTS=2 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
