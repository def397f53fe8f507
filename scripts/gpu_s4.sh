O=gpurun_out/s4; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x -rf --durations=10 > $O/gputests.log 2>&1
echo "pytest rc=$?"; tail -3 $O/gputests.log
rm -rf /dev/shm/vmsplat_test_c4 /dev/shm/vmsplat_test_shard_*
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
tail -1 $O/bench.log | cut -c1-300
timeout 600 python scripts/d2h_interf.py > $O/d2h.log 2>&1; tail -4 $O/d2h.log
