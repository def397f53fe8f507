set -x
timeout 600 python profiles/stage_bench.py --warm 10 --frames 20 > gpurun_out/stage_bin.txt 2>&1
VMSPLAT_TILE_SORT=radix timeout 600 python profiles/stage_bench.py --warm 10 --frames 20 > gpurun_out/stage_radix.txt 2>&1
