timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
VMSPLAT_PDL=0 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_nopdl.log 2>&1
