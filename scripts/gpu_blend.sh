set -x
timeout 1200 python -m pytest tests -m gpu -x -q -k "composite or c2 or render or overflow" 2>&1 | tail -3 > gpurun_out/gputests.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_f24.csv python profiles/profile_frames.py --warm 24 --frames 2 > gpurun_out/pf.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_f12.csv python profiles/profile_frames.py --warm 12 --frames 2 > gpurun_out/pf.log 2>&1
timeout 600 python profiles/e2e_modes.py > gpurun_out/e2e_modes.txt 2>&1
