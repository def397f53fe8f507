timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/gputests.log
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   -k regex:vis_raster --log-file gpurun_out/c3_raster.csv python profiles/profile_frames.py --config c3 --warm 12 --frames 1 > gpurun_out/c3pf.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   -k regex:vis_raster --log-file gpurun_out/c2_raster.csv python profiles/profile_frames.py --warm 12 --frames 1 > /dev/null 2>&1
