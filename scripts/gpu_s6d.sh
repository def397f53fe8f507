python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
cp paper_2506_19415_b200/libvmsplat_b200.so /tmp/step2.so
for rep in 1 2; do
for v in step2 step3; do
  [ $v = step2 ] && cp /tmp/step2.so paper_2506_19415_b200/libvmsplat_b200.so
  [ $v = step3 ] && cp .ab/libvmsplat_b200_step3.so paper_2506_19415_b200/libvmsplat_b200.so
  AB_TAG="$v 5-34" AB_TO=35 timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
  AB_TAG="$v 5-64" timeout 300 python scripts/value_ab.py 2>/dev/null | tail -1
done
done
cp .ab/libvmsplat_b200_step3.so paper_2506_19415_b200/libvmsplat_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "lane_lists or c2_whole" 2>&1 | tail -1
cp /tmp/step2.so paper_2506_19415_b200/libvmsplat_b200.so
for f in 12 25; do for v in step2 step3; do
  [ $v = step2 ] && cp /tmp/step2.so paper_2506_19415_b200/libvmsplat_b200.so
  [ $v = step3 ] && cp .ab/libvmsplat_b200_step3.so paper_2506_19415_b200/libvmsplat_b200.so
  echo "$v $(timeout 300 python profiles/blend_trace.py $f 2>/dev/null | head -1)"
done; done
cp /tmp/step2.so paper_2506_19415_b200/libvmsplat_b200.so
