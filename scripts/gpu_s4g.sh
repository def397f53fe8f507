# stream-priority A/B: front hi/lo x blend on caller/internal-hi stream
O=gpurun_out/s4g; mkdir -p $O
run() { timeout 600 env "$@" python bench.py --no-cpu-baseline > $O/b.log 2>&1
  echo "$* $(tail -1 $O/b.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["trajectory"]["value"], d["stages_ms"]["blend"])')"; }
for rep in 1 2; do
run VMSPLAT_FRONT_PRIO=1 VMSPLAT_BLEND_PRIO=0
run VMSPLAT_FRONT_PRIO=0 VMSPLAT_BLEND_PRIO=0
run VMSPLAT_FRONT_PRIO=0 VMSPLAT_BLEND_PRIO=1
run VMSPLAT_FRONT_PRIO=1 VMSPLAT_BLEND_PRIO=1
done
