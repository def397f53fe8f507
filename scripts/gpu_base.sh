set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/gputests.log gpurun_out/bench.log
