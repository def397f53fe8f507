set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "composite or c2_whole or overflow or output_modes" > gpurun_out/hot2_tests.log 2>&1
echo "hot tests rc=$?"
for v in "0 4096" "1 4096" "1 8192" "1 16384"; do
  set -- $v
  VMSPLAT_BLEND_HOT=$1 VMSPLAT_HOT_LEN=$2 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_hot_$1_$2.log 2>&1
  VMSPLAT_BLEND_HOT=$1 VMSPLAT_HOT_LEN=$2 timeout 600 python profiles/profile_frames.py --warm 25 --frames 1 --timing > gpurun_out/f25_hot_$1_$2.txt 2>&1
done
for v in "1 4096" "1 16384"; do
  set -- $v
  VMSPLAT_BLEND_HOT=$1 VMSPLAT_HOT_LEN=$2 timeout 900 python profiles/profile_frames.py --config c4 --warm 20 --frames 5 --timing > gpurun_out/c4_hot_$2.txt 2>&1
done
rm -rf /dev/shm/vmsplat_bench
tail -2 gpurun_out/hot2_tests.log
for v in 0_4096 1_4096 1_8192 1_16384; do python -c "import json;d=json.loads(open('gpurun_out/bench_hot_$v.log').read().strip().splitlines()[-1]);print('$v', d['value'], d['trajectory']['value'], d['e2e']['value'], d['stages_ms']['blend'])"; grep -E "^25 " gpurun_out/f25_hot_$v.txt | cut -c1-200; done
grep -E "^2[0-5] " gpurun_out/c4_hot_*.txt | cut -c1-250
