python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
  AB_TAG="default 5-34" AB_TO=35 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  for c in 70 100; do
    AB_TAG="carve$c 5-34" AB_TO=35 VMSPLAT_BLEND_CARVEOUT=$c timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  done
done
