O=gpurun_out/s4v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lane_lists or c2_whole or overlapped or composite or render_records or session_matches or 4k or overflow or resolution" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
for rep in 1 2; do
for nt in 256 128; do
  AB_TAG="nt$nt 5-64" VMSPLAT_BLEND_NT=$nt timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="nt$nt 5-34" AB_TO=35 VMSPLAT_BLEND_NT=$nt timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
for f in 12 25; do for nt in 256 128; do VMSPLAT_BLEND_NT=$nt timeout 300 python profiles/blend_trace.py $f 2>/dev/null | head -1; done; done
