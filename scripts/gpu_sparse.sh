# A/B of the sparse (splat-parallel) exact blend: parity on the session tests,
# then the C2 bench line with each variant
set -x
VMSPLAT_BLEND_SPARSE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "composite or render_records or session or c1 or c2_whole or overflow or output_modes or 4k or nothing" > gpurun_out/sparse_tests.log 2>&1
echo "sparse tests rc=$?"
for v in 0 1; do
  VMSPLAT_BLEND_SPARSE=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_sparse$v.log 2>&1
  VMSPLAT_BLEND_SPARSE=$v timeout 600 python profiles/profile_frames.py --warm 25 --frames 1 --trace > gpurun_out/trace25_sparse$v.txt 2>&1
  VMSPLAT_BLEND_SPARSE=$v timeout 600 python profiles/profile_frames.py --warm 12 --frames 1 --trace > gpurun_out/trace12_sparse$v.txt 2>&1
done
tail -3 gpurun_out/sparse_tests.log
for v in 0 1; do python -c "import json;d=json.loads(open('gpurun_out/bench_sparse$v.log').read().strip().splitlines()[-1]);print($v, d['value'], d['trajectory']['value'], d['e2e']['value'], d['stages_ms'])"; grep -E 'blend:|p50|p100' gpurun_out/trace25_sparse$v.txt gpurun_out/trace12_sparse$v.txt; done
