# device page table: unit/trace tests, session parity, and the C2 bench with
# the device table (VMSPLAT_DEVICE_TABLE=1) next to the host table
O=gpurun_out/r2; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dpt.py -m gpu -q -x > $O/dpt_tests.log 2>&1; echo "dpt tests rc=$?"; tail -15 $O/dpt_tests.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_host_$i.log 2>&1
  VMSPLAT_DEVICE_TABLE=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_dpt_$i.log 2>&1
done
for f in $O/bench_host_*.log $O/bench_dpt_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"], d["stages_ms"], d["clocks"]["sm_mhz"], d["host_wall_ms"])
except Exception as e:
    print(sys.argv[1], "ERR", e, open(sys.argv[1]).read()[-2000:])
PY
done
rm -rf /dev/shm/vmsplat_bench
