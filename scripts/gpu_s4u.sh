O=gpurun_out/s4u; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for f in 25 12; do
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:blend_k -c 1 -o $O/blend_f$f -f python profiles/profile_frames.py --warm $f --frames 1 > $O/ncu_f$f.log 2>&1
echo "ncu f$f rc=$?"
done
