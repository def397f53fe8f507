O=gpurun_out/s4n; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
AB_REPS=8 AB_VERBOSE=1 VMSPLAT_TRACE=1 timeout 600 python scripts/e2e_ab.py > $O/ab.log 2> $O/ab.err; cat $O/ab.log
grep -v "graph capture" $O/ab.err | grep vmsplat | tail -20
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
