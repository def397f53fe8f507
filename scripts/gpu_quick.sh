timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   -k regex:tile_prep --log-file gpurun_out/tp.csv python profiles/profile_frames.py --warm 12 --frames 1 > /dev/null 2>&1
VMSPLAT_TILE=16 timeout 600 python -m pytest tests -m gpu -x -q -k "c2_frames or session_matches or composite" 2>&1 | tail -2 > gpurun_out/gputests16.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
