set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 python profiles/frame_table.py --device > gpurun_out/ftab.txt 2>&1
VMSPLAT_GRAPHS=0 timeout 600 python profiles/frame_table.py --device > gpurun_out/ftab_ng.txt 2>&1
