set -x
timeout 600 python profiles/e2e_modes.py > gpurun_out/e2e_modes.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_f24.csv python profiles/profile_frames.py --warm 24 --frames 2 > gpurun_out/pf.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:blend_k -c 1 -o gpurun_out/blend2_f25 python profiles/profile_frames.py --warm 25 --frames 1 >> gpurun_out/pf.log 2>&1
