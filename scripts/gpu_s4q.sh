O=gpurun_out/s4q; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for f in 12 25 30 8; do timeout 300 python profiles/blend_trace.py $f 2>/dev/null | tee $O/trace_$f.txt | grep -v "^    "; done
