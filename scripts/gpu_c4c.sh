set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "streamed or c1_session" > gpurun_out/c4c_tests.log 2>&1
echo "tests rc=$?"
python profiles/profile_frames.py --config c4 --warm 20 --frames 5 --timing --trace > gpurun_out/c4c_f24.txt 2>&1
timeout 1200 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
echo "bench rc=$?"
rm -rf /dev/shm/vmsplat_bench
tail -3 gpurun_out/c4c_tests.log
grep -E "^2[0-5] |blend:|p50|p90|p99|p100|CTA start" gpurun_out/c4c_f24.txt | cut -c1-330
tail -c 1500 gpurun_out/bench_c4.log
