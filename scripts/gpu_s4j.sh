O=gpurun_out/s4j; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for e in 0 1; do
  VMSPLAT_EXP_NOHC=$e VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py d2h > $O/tl_d2h_$e.log 2>&1; grep fps $O/tl_d2h_$e.log
  python scripts/tl_summary.py $O/tl_d2h_$e.log
done
for k in 3 4; do
  VMSPLAT_SLOTS=$k timeout 600 python bench.py --no-cpu-baseline > $O/bench_s$k.log 2>&1
  echo "slots=$k $(tail -1 $O/bench_s$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
