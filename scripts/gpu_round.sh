# One lease: the GPU test suite, smoke(), the bench line (both arms), the
# launch list of the bench command and ncu --set full captures of the
# frame-12 render/visibility kernels and the frame-25 blend.  Logs under
# gpurun_out/r2/final/.
O=gpurun_out/r2/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
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
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:'blend|preprocess_k|dup_|tile_prep|radix|vis_|dpt_|scan|compact' -c 40 -o $O/full_f12 -f \
  python profiles/profile_frames.py --warm 12 --frames 1 > $O/ncu_f12.log 2>&1
echo "ncu f12 rc=$?"
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on \
  -k regex:blend_k -c 2 -o $O/full_f25_blend -f \
  python profiles/profile_frames.py --warm 25 --frames 1 > $O/ncu_f25.log 2>&1
echo "ncu f25 rc=$?"
timeout 600 python profiles/profile_frames.py --warm 5 --frames 30 --timing > $O/stages_5_34.txt 2>&1
rm -rf /dev/shm/vmsplat_bench
tail -1 $O/bench.log | cut -c1-300
tail -1 $O/bench_ref.log | cut -c1-300
