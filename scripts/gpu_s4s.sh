O=gpurun_out/s4s; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
for ll in 0 2 3; do
  AB_TAG="lanes$ll 5-64" VMSPLAT_LANE_LISTS=$ll timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="lanes$ll 5-34" AB_TO=35 VMSPLAT_LANE_LISTS=$ll timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
for f in 12 25; do VMSPLAT_LANE_LISTS=0 timeout 300 python profiles/blend_trace.py $f 2>/dev/null | head -1; VMSPLAT_LANE_LISTS=2 timeout 300 python profiles/blend_trace.py $f 2>/dev/null | head -1; done
