O=gpurun_out/s4y; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1; do
for k in 4 5 6; do
  AB_TAG="slots$k" VMSPLAT_SLOTS=$k timeout 300 python scripts/e2e_ab.py 2>/dev/null | tail -1
  AB_TAG="slots$k 5-34" AB_TO=35 VMSPLAT_SLOTS=$k timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
