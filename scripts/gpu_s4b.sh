# cross-frame overlap: parity tests, same-box A/B (VMSPLAT_OVERLAP=0/1), d2h interference, e2e timeline
O=gpurun_out/s4b; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "overlapped or c2_whole or output_modes or overflow or resolution or streamed" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/tests.log
for k in 1 0 1 0; do
  VMSPLAT_OVERLAP=$k timeout 600 python bench.py --no-cpu-baseline > $O/bench_ov$k.log 2>&1
  echo "overlap=$k $(tail -1 $O/bench_ov$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
timeout 300 python scripts/d2h_interf.py none d2h none > $O/d2h.log 2>&1; cat $O/d2h.log | grep fps
VMSPLAT_OVERLAP=0 timeout 300 python scripts/d2h_interf.py none d2h > $O/d2h_ov0.log 2>&1; cat $O/d2h_ov0.log | grep fps
timeout 300 python scripts/timeline_e2e.py > $O/tl.log 2>&1; grep -E "fps|GB" $O/tl.log
