O=gpurun_out/s5b; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x -k "radix or lane_lists or c2_whole or overlapped or binned or c3_frames or harness or shard" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
timeout 600 python bench.py --no-cpu-baseline > $O/bench.log 2>&1
tail -1 $O/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])'
