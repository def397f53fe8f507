# the whole GPU suite, smoke(), and the default bench line (both arms)
O=gpurun_out/r2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2700 python -m pytest tests -m gpu -q -rA --durations=25 > $O/gputests_full.log 2>&1
echo "pytest rc=$?"
rm -rf /dev/shm/vmsplat_test_c4 /dev/shm/vmsplat_test_shard_*
grep -E "passed|failed|FAILED|ERROR" $O/gputests_full.log | tail -15
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_full.log 2>&1; echo "bench rc=$?"
tail -1 $O/bench_full.log | cut -c1-400
timeout 900 python bench.py --impl reference --steps 30 --warmup 5 > $O/bench_ref_full.log 2>&1; echo "ref rc=$?"
tail -1 $O/bench_ref_full.log | cut -c1-300
rm -rf /dev/shm/vmsplat_bench
