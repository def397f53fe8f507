python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
for k in 1 0; do
  AB_TAG="small$k 5-34" AB_TO=35 VMSPLAT_RADIX_SMALL=$k timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="small$k 5-64" VMSPLAT_RADIX_SMALL=$k timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
