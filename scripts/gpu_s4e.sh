# 3 frame slots: tests, slot-count A/B, e2e timeline
O=gpurun_out/s4e; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dpt.py tests/test_gpu_parity.py tests/test_harness.py tests/test_gpu_scale.py -m gpu -q -x -k "dpt or device_table or overlapped or c2_whole or session or harness or shard or pipelin or output" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
for k in 3 2 4 3; do
  VMSPLAT_SLOTS=$k timeout 600 python bench.py --no-cpu-baseline > $O/bench_s$k.log 2>&1
  echo "slots=$k $(tail -1 $O/bench_s$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
timeout 300 python scripts/timeline_e2e.py > $O/tl_e2e.log 2>&1; grep -E "fps|GB" $O/tl_e2e.log
