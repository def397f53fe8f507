# device timeline under a concurrent image copy, 3 slots
O=gpurun_out/s4i; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for m in none d2h h2d_unrel; do
  VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py $m > $O/tl_$m.log 2>&1; grep fps $O/tl_$m.log
done
VMSPLAT_TRACE=2 timeout 300 python scripts/timeline_e2e.py > $O/tl_e2e.log 2>&1; grep -E "fps|GB" $O/tl_e2e.log
