timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/gputests.log
timeout 600 python profiles/bvh_bench.py > gpurun_out/bvh_bench.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bvh_nearest -c 1 -o gpurun_out/bvh_full python profiles/bvh_bench.py --points 500000 --cpu-points 100 > /dev/null 2>&1
