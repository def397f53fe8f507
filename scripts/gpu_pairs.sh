timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/gputests.log
for pv in 0 1; do for f in 12 25 50; do
VMSPLAT_BLEND_PAIRS=$pv timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
   -k regex:blend --log-file gpurun_out/bl_p${pv}_f$f.csv python profiles/profile_frames.py --warm $f --frames 1 > /dev/null 2>&1
done; done
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1
