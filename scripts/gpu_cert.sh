O=gpurun_out/r2; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -s -k "certified or session_matches_reference or composite" > $O/cert_tests.log 2>&1; echo "cert tests rc=$?"
grep -E "certified fast|passed|failed|Error|assert" $O/cert_tests.log | tail -12
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --fast > $O/bench_fast_$i.log 2>&1
done
for f in $O/bench_fast_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["stages_ms"], d["clocks"]["sm_mhz"])
except Exception as e:
    print(sys.argv[1], "ERR", e, open(sys.argv[1]).read()[-2000:])
PY
done
timeout 600 python profiles/profile_frames.py --fast --warm 5 --frames 30 --timing > $O/stages_5_34_fast.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:'blend' -c 4 -o $O/full_fast_f25 -f python profiles/profile_frames.py --fast --warm 25 --frames 1 > $O/ncu_fast.log 2>&1
echo "ncu rc=$?"
rm -rf /dev/shm/vmsplat_bench
