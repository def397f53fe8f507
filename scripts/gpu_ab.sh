# A/B of the working tree's library against .ab/libvmsplat_b200_old.so on one
# box (C2 bench, two runs each, interleaved), after the parity subset
O=gpurun_out/r2; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "${AB_TESTS:-c2_whole or session_matches or composite or certified}" > $O/ab_parity.log 2>&1; echo "parity rc=$?"; tail -1 $O/ab_parity.log
cp paper_2506_19415_b200/libvmsplat_b200.so /tmp/new.so
for i in 1 2; do
  cp /tmp/new.so paper_2506_19415_b200/libvmsplat_b200.so
  timeout 600 python bench.py --no-cpu-baseline > $O/ab_new_$i.log 2>&1
  cp .ab/libvmsplat_b200_old.so paper_2506_19415_b200/libvmsplat_b200.so
  timeout 600 python bench.py --no-cpu-baseline > $O/ab_old_$i.log 2>&1
done
cp /tmp/new.so paper_2506_19415_b200/libvmsplat_b200.so
for f in $O/ab_new_*.log $O/ab_old_*.log; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], d["value"], d["e2e"]["value"], d["stages_ms"]["blend"], d["stages_ms"]["device_frame"])
PY
done
rm -rf /dev/shm/vmsplat_bench
