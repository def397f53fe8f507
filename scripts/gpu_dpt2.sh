O=gpurun_out/r2; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dpt.py -m gpu -q -x > $O/dpt_tests2.log 2>&1; echo "dpt tests rc=$?"; tail -2 $O/dpt_tests2.log
for cfg in c4 c2; do
  VMSPLAT_DEVICE_TABLE=1 timeout 1500 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}_dpt2.log 2>&1; echo "$cfg dpt rc=$?"
  VMSPLAT_DEVICE_TABLE=0 timeout 1500 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}_host2.log 2>&1; echo "$cfg host rc=$?"
done
for f in $O/bench_*2.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d["e2e"]["value"], d.get("e2e_sync",{}).get("value"), d["stages_ms"]["visibility"], d["stages_ms"]["device_frame"], d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "ERR", e, open(sys.argv[1]).read()[-1500:])
PY
done
rm -rf /dev/shm/vmsplat_bench
