O=gpurun_out/s5d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_harness.py -m gpu -q -x -k "streamed or pipelined or overlapped or c1_session" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
for k in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench$k.log 2>&1
  tail -1 $O/bench$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"])'
done
rm -rf /dev/shm/vmsplat_bench
timeout 2400 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.log 2>&1; echo "c4 rc=$?"
tail -1 $O/bench_c4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"], d["upload"])'
