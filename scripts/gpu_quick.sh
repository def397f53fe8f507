timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 python profiles/e2e_modes.py > gpurun_out/e2e_modes.txt 2>&1
