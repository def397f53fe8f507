# device-memory required list for the device page table: tests, interference, bench
O=gpurun_out/s4d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dpt.py tests/test_gpu_parity.py -m gpu -q -x -k "dpt or device_table or overlapped or c2_whole or session" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
for m in none d2h h2d_unrel; do
  VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py $m > $O/tl_$m.log 2>&1; grep fps $O/tl_$m.log
done
for k in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench$k.log 2>&1
  echo "bench $(tail -1 $O/bench$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
timeout 300 python scripts/timeline_e2e.py > $O/tl_e2e.log 2>&1; grep -E "fps|GB" $O/tl_e2e.log
