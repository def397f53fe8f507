timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
VMSPLAT_HOT=0 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_h0.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_h1.log 2>&1
VMSPLAT_HOT=0 timeout 600 python profiles/frame_table.py > gpurun_out/ft_h0.txt 2>&1
timeout 600 python profiles/frame_table.py > gpurun_out/ft_h1.txt 2>&1
