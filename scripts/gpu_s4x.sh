O=gpurun_out/s4x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lane_lists or c2_whole or overlapped or composite or render_records or session_matches or certified" > $O/tests.log 2>&1
echo "pytest rc=$?"; tail -2 $O/tests.log
cp paper_2506_19415_b200/libvmsplat_b200.so /tmp/new.so
for rep in 1 2; do
for v in old new; do
  cp .ab/libvmsplat_b200_old.so paper_2506_19415_b200/libvmsplat_b200.so
  [ $v = new ] && cp /tmp/new.so paper_2506_19415_b200/libvmsplat_b200.so
  AB_TAG="$v 5-64" timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="$v 5-34" AB_TO=35 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
cp /tmp/new.so paper_2506_19415_b200/libvmsplat_b200.so
for f in 12 25; do timeout 300 python profiles/blend_trace.py $f 2>/dev/null | head -1; done
timeout 600 ncu --profile-from-start off --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,gpu__time_duration.sum --clock-control none \
  -k regex:blend_k -c 1 python profiles/profile_frames.py --warm 25 --frames 1 2>&1 | grep -E "conflicts|wavefronts|duration" 
