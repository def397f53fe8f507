# Round-1 evidence (final): bench JSON, launch list of the bench command, ncu
# --set full of the render + visibility kernels of frame 12 and the blend of
# frame 25.
set -x
mkdir -p gpurun_out/prof
timeout 900 python bench.py > gpurun_out/prof/bench.json.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/prof/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/prof/bench_under_ncu.log 2>&1
timeout 1500 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"blend_k|preprocess_k|radix_onesweep_k|dup_emit_k|vis_raster_k|tile_prep_k|dup_count_k|vis_back_k" -c 16 \
  -o gpurun_out/prof/full_f12 python profiles/profile_frames.py --warm 12 --frames 1 > gpurun_out/prof/full_f12.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:"blend_k" -c 1 -o gpurun_out/prof/full_f25_blend python profiles/profile_frames.py --warm 25 --frames 1 > gpurun_out/prof/full_f25.log 2>&1
