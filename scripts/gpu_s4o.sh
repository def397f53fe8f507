O=gpurun_out/s4o; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_dpt.py tests/test_gpu_parity.py tests/test_harness.py tests/test_gpu_scale.py tests/test_reference_suite.py -m gpu -q -x -k "dpt or device_table or overlapped or c2_whole or session or harness or shard or pipelin or output or c4" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
AB_REPS=8 AB_VERBOSE=1 timeout 600 python scripts/e2e_ab.py > $O/ab.log 2>&1; tail -1 $O/ab.log
for k in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench$k.log 2>&1
  echo "bench $(tail -1 $O/bench$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
