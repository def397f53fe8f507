for k in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$k.log 2>&1; done
