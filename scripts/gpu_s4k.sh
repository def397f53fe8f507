O=gpurun_out/s4k; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for m in none d2h d2h_chunk8 d2h_sm; do
  VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py $m > $O/tl_$m.log 2>&1; grep fps $O/tl_$m.log; tail -2 $O/tl_$m.log | grep -i error
  python scripts/tl_summary.py $O/tl_$m.log
done
