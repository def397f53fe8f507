python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
for b in 4 8 16; do
  AB_TAG="bands$b" VMSPLAT_D2H_BANDS=$b timeout 300 python scripts/e2e_ab.py 2>/dev/null | tail -1
done
done
