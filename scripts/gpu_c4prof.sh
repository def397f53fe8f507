# C4 (tmpfs scene): per-stage times + blend trace of a slow frame, ncu of the
# visibility kernels and the blend of that frame
set -x
python profiles/profile_frames.py --config c4 --warm 20 --frames 6 --timing --trace > gpurun_out/c4_stages.txt 2>&1
ncu --profile-from-start off --set full --clock-control none -k regex:'vis_|radix' -c 12 -o gpurun_out/c4_vis -f python profiles/profile_frames.py --config c4 --warm 20 --frames 1 > gpurun_out/c4_ncu_vis.log 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python profiles/profile_frames.py --config c4 --warm 20 --frames 2 > /dev/null 2>&1
rm -rf /dev/shm/vmsplat_bench
tail -30 gpurun_out/c4_stages.txt
