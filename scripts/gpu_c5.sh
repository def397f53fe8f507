timeout 2400 python bench.py --config c3 --width 3840 --height 2160 --no-cpu-baseline --steps 20 > gpurun_out/bench_c5.log 2>&1
timeout 2400 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3.log 2>&1
