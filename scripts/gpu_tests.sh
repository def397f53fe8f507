# full GPU test suite + the default bench line (one lease)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=15 ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1
echo "pytest rc=$?"
rm -rf /dev/shm/vmsplat_test_c4 /dev/shm/vmsplat_test_shard_*
if [ -z "$NO_BENCH" ]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
  timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
fi
tail -25 gpurun_out/gputests.log
