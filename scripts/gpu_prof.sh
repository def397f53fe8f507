# per-kernel stage bench + ncu launch list + full capture of the top kernels
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene to /tmp
timeout 600 python profiles/stage_bench.py --warm 12 --frames 10 > gpurun_out/stage_bench.txt 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python profiles/profile_frames.py > gpurun_out/pf.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
   -k regex:"blend_k|radix_onesweep_k|dup_emit_k|preprocess_k" -c 6 -o gpurun_out/full python profiles/profile_frames.py > gpurun_out/full.log 2>&1
python profiles/launch_summary.py gpurun_out/launches.csv > gpurun_out/launch_summary.txt 2>&1
