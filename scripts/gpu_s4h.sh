# full suite + smoke + bench (trajectory spike diagnosis)
O=gpurun_out/s4h; mkdir -p $O
rm -rf /dev/shm/vmsplat_bench
VMSPLAT_TRACE=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench1.log 2> $O/bench1.err
tail -1 $O/bench1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["trajectory"])'
timeout 600 python bench.py --no-cpu-baseline > $O/bench2.log 2>&1
tail -1 $O/bench2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["trajectory"])'
timeout 1500 python -m pytest tests -m gpu -q -x -rf --durations=5 > $O/gputests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
