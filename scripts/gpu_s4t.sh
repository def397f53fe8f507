O=gpurun_out/s4t; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py none > $O/tl_none.log 2>&1; grep fps $O/tl_none.log
python scripts/tl_summary.py $O/tl_none.log --frames
VMSPLAT_OVERLAP=0 VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py none > $O/tl_serial.log 2>&1; grep fps $O/tl_serial.log
python scripts/tl_summary.py $O/tl_serial.log --frames
