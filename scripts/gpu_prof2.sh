# ncu of the F2/F3 kernels, and the C3 / C4 bench lines with the device and
# the host page table
O=gpurun_out/r2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lod_page_k -c 1 \
  -o $O/full_lod -f python profiles/lod_bench.py --pages 296 --reps 1 --cpu-pages 0 > $O/ncu_lod.log 2>&1
echo "ncu lod rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:dpt_ -c 4 -o $O/full_dpt -f python profiles/profile_frames.py --warm 12 --frames 2 > $O/ncu_dpt.log 2>&1
echo "ncu dpt rc=$?"
timeout 900 python profiles/profile_frames.py --warm 5 --frames 30 --timing > $O/stages_5_34_dpt.txt 2>&1
for cfg in c3 c4; do
  timeout 1500 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}_dpt.log 2>&1; echo "$cfg dpt rc=$?"
  VMSPLAT_DEVICE_TABLE=0 timeout 1500 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}_host.log 2>&1; echo "$cfg host rc=$?"
done
for f in $O/bench_c3_*.log $O/bench_c4_*.log; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], d["value"], d["e2e"]["value"], d.get("e2e_sync",{}).get("value"), d["stages_ms"], d["clocks"]["sm_mhz"], d.get("upload"))
except Exception as e:
    print(sys.argv[1], "ERR", e, open(sys.argv[1]).read()[-1500:])
PY
done
rm -rf /dev/shm/vmsplat_bench /dev/shm/vmsplat_*
