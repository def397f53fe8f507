# the whole -m gpu suite and smoke() on the current code
O=gpurun_out/r2/final3; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q -rf --durations=10 > $O/gputests_last.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" $O/gputests_last.log | tail -2
rm -rf /dev/shm/vmsplat_test_c4 /dev/shm/vmsplat_test_shard_*
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_last.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke_last.log
