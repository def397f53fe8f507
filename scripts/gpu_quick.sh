timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
   -k regex:preprocess --log-file gpurun_out/pre.csv python profiles/profile_frames.py --warm 12 --frames 1 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
