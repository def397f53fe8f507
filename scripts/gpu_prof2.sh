set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gputests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_f24.csv python profiles/profile_frames.py --warm 24 --frames 2 > gpurun_out/pf.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_f12.csv python profiles/profile_frames.py --warm 12 --frames 2 >> gpurun_out/pf.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:blend_k -c 1 -o gpurun_out/blend_f25 python profiles/profile_frames.py --warm 25 --frames 1 >> gpurun_out/pf.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"radix_onesweep_k|dup_emit_k|ranges_k|radix_hist_k|preprocess_k" -c 12 -o gpurun_out/tiles_f12 python profiles/profile_frames.py --warm 12 --frames 1 >> gpurun_out/pf.log 2>&1
