timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 900 python bench.py --no-cpu-baseline --upload-mode 2 > gpurun_out/bench_stream.log 2>&1
