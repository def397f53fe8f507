python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for rep in 1 2; do
  for u in 0 1; do
    AB_TAG="upload$u" AB_UPLOAD=$u timeout 300 python scripts/e2e_ab.py 2>/dev/null | tail -1
    AB_TAG="upload$u 5-34" AB_TO=35 AB_UPLOAD=$u timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  done
done
