free -g | head -2
timeout 1500 python scripts/c4_probe.py > gpurun_out/c4_probe.log 2>&1
echo rc=$?
free -g | head -2
rm -rf /dev/shm/vmsplat_bench
tail -5 gpurun_out/c4_probe.log
