timeout 600 python bench.py --no-cpu-baseline --upload-mode 0 > gpurun_out/bench_u0.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --upload-mode 1 > gpurun_out/bench_u1.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --upload-mode 2 > gpurun_out/bench_u2.log 2>&1
