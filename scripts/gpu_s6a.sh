O=gpurun_out/s6a; mkdir -p $O
VMSPLAT_TILE_SORT1=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2_whole or overlapped or composite or render_records or session_matches or c1_session or 4k or overflow or resolution" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log; grep -E "Error|assert" $O/tests.log | head -5
for rep in 1 2; do
for k in 0 1; do
  AB_TAG="sort1=$k 5-34" AB_TO=35 VMSPLAT_TILE_SORT1=$k timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="sort1=$k 5-64" VMSPLAT_TILE_SORT1=$k timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
VMSPLAT_TILE_SORT1=1 timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -k regex:"digit_scatter|radix_onesweep|dup_emit" python profiles/profile_frames.py --warm 12 --frames 1 2>&1 | grep -E "digit_scatter|onesweep|dup_emit|duration" | head -20
