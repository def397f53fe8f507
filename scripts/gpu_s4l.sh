O=gpurun_out/s4l; mkdir -p $O
for rep in 1 2; do
for k in 1 8 32; do
  VMSPLAT_D2H_BANDS=$k timeout 600 python bench.py --no-cpu-baseline > $O/bench_b$k.log 2>&1
  echo "bands=$k $(tail -1 $O/bench_b$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
done
