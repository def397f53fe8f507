# device-mode timeline (front end / blend start), bench with the pre-sized output pool
O=gpurun_out/s4f; mkdir -p $O
for k in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench$k.log 2>&1
  echo "bench $(tail -1 $O/bench$k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"])')"
done
VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py none > $O/tl_none.log 2>&1; grep fps $O/tl_none.log
timeout 300 python scripts/timeline_e2e.py > $O/tl_e2e.log 2>&1; grep -E "fps|GB" $O/tl_e2e.log
