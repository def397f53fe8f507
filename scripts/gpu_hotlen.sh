# hot-tile blend threshold sweep on C2 (frames 5-34)
O=gpurun_out/r2; mkdir -p $O
for h in 32768 8192 6144 4096 3072; do
  VMSPLAT_HOT_LEN=$h timeout 600 python bench.py --no-cpu-baseline > $O/bench_hot_$h.log 2>&1
  python - "$O/bench_hot_$h.log" $h <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("hot_len", sys.argv[2], d["value"], d["e2e"]["value"], d["stages_ms"]["blend"])
PY
done
for h in 32768 4096; do
  VMSPLAT_HOT_LEN=$h timeout 600 python profiles/profile_frames.py --warm 25 --frames 1 --timing --trace > $O/trace25_hot_$h.txt 2>&1
  grep -E "^25 |blend:" $O/trace25_hot_$h.txt | cut -c1-250
done
rm -rf /dev/shm/vmsplat_bench
