import ctypes, os, sys, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_19415_b200 import scenegen
from paper_2506_19415_b200.scene_io import read_scene
rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
rt.cudaGetErrorString.restype = ctypes.c_char_p
lay = scenegen.C4
d = "/dev/shm/vmsplat_bench"; os.makedirs(d, exist_ok=True)
p = os.path.join(d, "c4.vms")
t = time.time(); scenegen.write_city(p, lay); print("gen", time.time() - t, flush=True)
os.system("grep -E 'MemFree|MemAvailable|Shmem:|Mlocked|Unevictable' /proc/meminfo")
os.system("grep -E '^Node|present|managed|  free ' /proc/zoneinfo | head -40")
sc = read_scene(p, mmap_gaussians=True)
mm = np.memmap(p, dtype="<f4", mode="r+", offset=sc.gaus_offset, shape=sc.gaussians.shape)
base = mm.ctypes.data & ~4095
end = (mm.ctypes.data + mm.nbytes + 4095) & ~4095
t = time.time()
e = rt.cudaHostRegister(ctypes.c_void_p(base), ctypes.c_size_t(end - base), ctypes.c_uint(11))
print("whole", e, rt.cudaGetErrorString(e).decode(), time.time() - t, flush=True)
if e == 0:
    rt.cudaHostUnregister(ctypes.c_void_p(base))
rt.cudaGetLastError()
chunk = 4 << 30
ok = 0
t = time.time()
regs = []
for a in range(base, end, chunk):
    b = min(end, a + chunk)
    e = rt.cudaHostRegister(ctypes.c_void_p(a), ctypes.c_size_t(b - a), ctypes.c_uint(11))
    if e:
        print("chunk fail at", (a - base) >> 30, "GB", rt.cudaGetErrorString(e).decode(), flush=True)
        rt.cudaGetLastError()
        break
    regs.append(a); ok += b - a
print("chunked ok GB", ok >> 30, time.time() - t, flush=True)
os.system("grep -E 'MemFree|MemAvailable|Shmem:|Mlocked|Unevictable' /proc/meminfo")
for a in regs:
    rt.cudaHostUnregister(ctypes.c_void_p(a))
os.unlink(p)
