python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
  AB_TAG="base 5-34" AB_TO=35 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="front_prio0 5-34" AB_TO=35 VMSPLAT_FRONT_PRIO=0 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="vis_prio0 5-34" AB_TO=35 VMSPLAT_VIS_PRIO=0 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="pre1 5-34" AB_TO=35 VMSPLAT_PRE_PER_SM=1 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="emit2 5-34" AB_TO=35 VMSPLAT_EMIT_PER_SM=2 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
