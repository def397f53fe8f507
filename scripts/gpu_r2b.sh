# LOD GPU tests, the hot-tile gate (C4 parity + hot-tile test), the bench line,
# then compute-sanitizer memcheck/racecheck/synccheck (scripts/gpu_sanitize.sh)
O=gpurun_out/r2; mkdir -p $O
timeout 900 python -m pytest tests/test_lod.py -m gpu -q > $O/lod_tests.log 2>&1; echo "lod tests rc=$?"; tail -2 $O/lod_tests.log
timeout 1500 python -m pytest tests/test_gpu_scale.py -m gpu -q -k "c4 or hot" > $O/hot_tests.log 2>&1; echo "hot tests rc=$?"; tail -2 $O/hot_tests.log
rm -rf /dev/shm/vmsplat_test_c4
timeout 600 python bench.py --no-cpu-baseline > $O/bench_gate.log 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('$O/bench_gate.log').read().strip().splitlines()[-1]);print(d['value'],d['e2e']['value'],d['stages_ms'],d['clocks'])"
bash scripts/gpu_sanitize.sh
mkdir -p $O/sanitize && cp gpurun_out/sanitize/*.log $O/sanitize/ 2>/dev/null
rm -rf /dev/shm/vmsplat_bench
