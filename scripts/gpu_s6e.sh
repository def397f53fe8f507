O=gpurun_out/s6e; mkdir -p $O
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 $O/bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e_sync"]["value"], d["trajectory"]["value"], d["gpu_launches"], d["cpu_baseline"]["value"], d["clocks"])'
tail -1 $O/bench_ref.log | cut -c1-300
