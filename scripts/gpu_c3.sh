timeout 2400 python bench.py --config c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
