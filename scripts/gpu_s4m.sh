O=gpurun_out/s4m; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
for k in 1 4 8 16; do
  AB_TAG=bands$k VMSPLAT_D2H_BANDS=$k timeout 300 python scripts/e2e_ab.py 2>/dev/null | tail -1
done
done
