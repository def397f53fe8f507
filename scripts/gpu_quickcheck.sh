timeout 300 python -m pytest tests -m gpu -x -q -k "session_matches or c2_frames or composite" 2>&1 | tail -2 > gpurun_out/gputests.log
for k in 1 2; do timeout 240 python bench.py --no-cpu-baseline > gpurun_out/bench_$k.log 2>&1; done
