timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_f12.csv python profiles/profile_frames.py --warm 12 --frames 2 > gpurun_out/pf.log 2>&1
