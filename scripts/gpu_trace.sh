timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
timeout 300 python profiles/blend_trace.py 25 > gpurun_out/trace25.txt 2>&1
timeout 300 python profiles/blend_trace.py 12 > gpurun_out/trace12.txt 2>&1
timeout 300 python profiles/blend_trace.py 50 > gpurun_out/trace50.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
