O=gpurun_out/r2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_dpt.py -m gpu -q -x 2>&1 | tail -1
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline > $O/ab2_dpt_$i.log 2>&1
  VMSPLAT_DEVICE_TABLE=0 timeout 600 python bench.py --no-cpu-baseline > $O/ab2_host_$i.log 2>&1
done
for c in 8 16; do
  VMSPLAT_COPY_THREADS=$c timeout 1500 python bench.py --config c4 --no-cpu-baseline > $O/c4_threads_$c.log 2>&1
done
for f in $O/ab2_*.log $O/c4_threads_*.log; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["stages_ms"]["visibility"], d["stages_ms"]["copy"], d.get("upload",{}).get("gbs"))
PY
done
rm -rf /dev/shm/vmsplat_bench
