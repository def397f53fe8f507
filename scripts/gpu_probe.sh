free -g; df -h /tmp /dev/shm /root; nproc; lscpu | head -20; cat /proc/meminfo | head -5; ulimit -l; nvidia-smi topo -m | head -5
python - <<'PY' > gpurun_out/probe_pcie.txt 2>&1
import torch, time
torch.cuda.init()
for mb in (256,):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device='cuda')
    s = torch.cuda.Stream()
    best_h2d = best_d2h = 0
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(); d.copy_(h, non_blocking=True); e1.record()
        e1.synchronize(); best_h2d = max(best_h2d, n / e0.elapsed_time(e1) / 1e6)
        with torch.cuda.stream(s):
            e0.record(); h.copy_(d, non_blocking=True); e1.record()
        e1.synchronize(); best_d2h = max(best_d2h, n / e0.elapsed_time(e1) / 1e6)
    print("h2d GB/s", best_h2d, "d2h GB/s", best_d2h)
PY
cat gpurun_out/probe_pcie.txt
