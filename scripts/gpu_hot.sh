# hot-tile blend: parity (C2 trajectory incl. the vanishing-point frames, C3,
# C4 windows), then A/B of the C2 bench and C4 stage times
set -x
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -m gpu -x -k "composite or render_records or session or c1 or c2_whole or overflow or output_modes or 4k or c3 or c4 or nothing" > gpurun_out/hot_tests.log 2>&1
echo "hot tests rc=$?"
for v in 0 1; do
  VMSPLAT_BLEND_HOT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_hot$v.log 2>&1
  VMSPLAT_BLEND_HOT=$v timeout 600 python profiles/profile_frames.py --warm 25 --frames 1 --trace --timing > gpurun_out/trace25_hot$v.txt 2>&1
done
VMSPLAT_BLEND_HOT=1 timeout 900 python profiles/profile_frames.py --config c4 --warm 20 --frames 5 --timing > gpurun_out/c4_hot.txt 2>&1
rm -rf /dev/shm/vmsplat_bench /dev/shm/vmsplat_test_c4
tail -3 gpurun_out/hot_tests.log
for v in 0 1; do python -c "import json;d=json.loads(open('gpurun_out/bench_hot$v.log').read().strip().splitlines()[-1]);print($v, d['value'], d['trajectory']['value'], d['e2e']['value'], d['stages_ms'])"; grep -E "^25 " gpurun_out/trace25_hot$v.txt | cut -c1-300; done
grep -E "^2[0-5] " gpurun_out/c4_hot.txt | cut -c1-300
