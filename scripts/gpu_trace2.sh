timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
for f in 12 25 50; do timeout 300 python profiles/blend_trace.py $f > gpurun_out/trace${f}_a.txt 2>&1; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
