O=gpurun_out/s4p; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
for ns in 0 32 128 512; do
  AB_TAG="sleep$ns 5-64" VMSPLAT_LB_SLEEP=$ns timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="sleep$ns 5-34" AB_TO=35 VMSPLAT_LB_SLEEP=$ns timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
for rep in 1 2; do
for t in 32 16; do
  AB_TAG="tile$t 5-64" VMSPLAT_TILE=$t timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="tile$t 5-34" AB_TO=35 VMSPLAT_TILE=$t timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
