timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   -k regex:"vis_" --log-file gpurun_out/vis12.csv python profiles/profile_frames.py --warm 12 --frames 1 > /dev/null 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   -k regex:"vis_" --log-file gpurun_out/c3vis.csv python profiles/profile_frames.py --config c3 --warm 12 --frames 1 > gpurun_out/c3pf.log 2>&1
timeout 2400 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/bench_c3.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
