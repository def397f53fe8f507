# Final capture, last code of round 2 (4 slots, radix grid cap): suite, smoke, both arms, launch list, C3/4K/C4 (WITH_SAN / WITH_FULL add sanitizers / ncu full captures)
O=gpurun_out/r2/final3; mkdir -p $O/sanitize
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
CS="compute-sanitizer --print-limit 50 --error-exitcode 9"
if [ -n "$WITH_SAN" ]; then
timeout 1200 $CS --tool memcheck python profiles/profile_frames.py --warm 24 --frames 3 > $O/sanitize/frames_memcheck.log 2>&1; echo "frames memcheck rc=$?"
timeout 1200 $CS --tool racecheck python profiles/profile_frames.py --warm 24 --frames 2 > $O/sanitize/frames_racecheck.log 2>&1; echo "frames racecheck rc=$?"
timeout 1200 $CS --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "overlapped and None" > $O/sanitize/overlap_memcheck.log 2>&1; echo "overlap memcheck rc=$?"
fi
if [ -z "$NO_TESTS" ]; then
  timeout 2700 python -m pytest tests -m gpu -q -rA --durations=25 > $O/gputests.log 2>&1
  echo "pytest rc=$?"
  rm -rf /dev/shm/vmsplat_test_c4 /dev/shm/vmsplat_test_shard_*
  grep -E "passed|failed" $O/gputests.log | tail -2
fi
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_ncu.log 2>&1
echo "ncu launches rc=$?"
if [ -n "$WITH_FULL" ]; then timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:'blend|preprocess_k|dup_|tile_prep|radix|vis_|dpt_|scan|compact|hot_list' -c 40 -o $O/full_f12 -f \
  python profiles/profile_frames.py --warm 12 --frames 1 > $O/ncu_f12.log 2>&1
echo "ncu f12 rc=$?"; fi
if [ -n "$WITH_FULL" ]; then timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:blend_k -c 1 -o $O/full_f25_blend -f \
  python profiles/profile_frames.py --warm 25 --frames 1 > $O/ncu_f25.log 2>&1
echo "ncu f25 rc=$?"; fi
timeout 600 python profiles/profile_frames.py --warm 5 --frames 30 --timing > $O/stages_5_34.txt 2>&1
VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py none > $O/tl_device.log 2>&1
python scripts/tl_summary.py $O/tl_device.log --frames > $O/tl_device_summary.txt
rm -rf /dev/shm/vmsplat_bench
tail -1 $O/bench.log | cut -c1-300
tail -1 $O/bench_ref.log | cut -c1-300
if [ -z "$NO_BIG" ]; then
timeout 1200 python bench.py --config c3 --no-cpu-baseline > $O/bench_c3.log 2>&1; echo "c3 rc=$?"; tail -1 $O/bench_c3.log | cut -c1-200
timeout 900 python bench.py --config c3 --width 3840 --height 2160 --no-cpu-baseline > $O/bench_c3_4k.log 2>&1; echo "c3 4k rc=$?"; tail -1 $O/bench_c3_4k.log | cut -c1-200
rm -rf /dev/shm/vmsplat_bench
timeout 2400 python bench.py --config c4 --no-cpu-baseline > $O/bench_c4.log 2>&1; echo "c4 rc=$?"; tail -1 $O/bench_c4.log | cut -c1-200
rm -rf /dev/shm/vmsplat_bench
fi
