python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
  for h in 1 0; do
    AB_TAG="hot$h 5-34" AB_TO=35 VMSPLAT_BLEND_HOT=$h timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  done
done
