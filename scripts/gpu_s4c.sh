# visibility latency under a concurrent image copy (timeline per mode)
O=gpurun_out/s4c; mkdir -p $O
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1   # writes the scene
for m in none d2h h2d_unrel d2d_unrel; do
  VMSPLAT_TRACE=2 timeout 300 python scripts/d2h_interf.py $m > $O/tl_$m.log 2>&1; grep fps $O/tl_$m.log
done
nvidia-smi -q | grep -i -A3 "copy\|PCIe\|Link Width\|Generation" | head -40 > $O/smi.txt
python - <<'PY' > $O/props.txt 2>&1
import torch
p = torch.cuda.get_device_properties(0)
print(p)
from cuda import cudart
err, v = cudart.cudaDeviceGetAttribute(cudart.cudaDeviceAttr.cudaDevAttrAsyncEngineCount, 0)
print("asyncEngineCount", v)
PY
cat $O/props.txt
