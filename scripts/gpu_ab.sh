# LOD kernel parity + measurement, and an A/B of the C2 bench: this build
# (hot-tile path on / off) vs the round-1 build (.ab_r1, same page-upload
# call), two runs each, interleaved.
O=gpurun_out/r2; mkdir -p $O
timeout 900 python -m pytest tests/test_lod.py -m gpu -q -x > $O/lod_tests.log 2>&1; echo "lod tests rc=$?"
tail -3 $O/lod_tests.log
timeout 900 python profiles/lod_bench.py --pages 1000 > $O/lod_bench.json 2>$O/lod_bench.err; echo "lod bench rc=$?"
cat $O/lod_bench.json; tail -3 $O/lod_bench.err
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/ab_hot1_$i.log 2>&1
  VMSPLAT_BLEND_HOT=0 timeout 600 python bench.py --no-cpu-baseline > $O/ab_hot0_$i.log 2>&1
  (cd .ab_r1 && timeout 600 python bench.py --no-cpu-baseline) > $O/ab_r1_$i.log 2>&1
done
for f in $O/ab_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d.get("e2e",{}).get("value"), d.get("stages_ms"), d.get("clocks"))
except Exception as e:
    print(sys.argv[1], "ERR", e)
PY
done
rm -rf /dev/shm/vmsplat_bench /tmp/vmsplat_bench
