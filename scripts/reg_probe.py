import ctypes, os, numpy as np, mmap
rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
rt.cudaGetErrorString.restype = ctypes.c_char_p
def attr(a):
    v = ctypes.c_int(); e = rt.cudaDeviceGetAttribute(ctypes.byref(v), a, 0); return (e, v.value)
# 99 HostRegisterSupported? use known enums: cudaDevAttrHostRegisterSupported=99, ReadOnly=113, CanUseHostPointerForRegisteredMem=91, PageableMemoryAccess=88
for name, a in (("HostRegisterSupported", 99), ("HostRegisterReadOnlySupported", 113),
                ("CanUseHostPointerForRegisteredMem", 91), ("PageableMemoryAccess", 88),
                ("PageableMemoryAccessUsesHostPageTables", 100)):
    print(name, attr(a))
for d in ("/dev/shm", "/tmp"):
    p = os.path.join(d, "regprobe.bin")
    with open(p, "wb") as fh:
        fh.write(b"\0" * 64 + np.arange(1 << 22, dtype=np.float32).tobytes())
    for mode, flags in (("r", 1 | 2 | 8), ("r", 1 | 2), ("r+", 1 | 2), ("r+", 1 | 2 | 8), ("r", 8), ("r", 2|8)):
        mm = np.memmap(p, dtype=np.float32, mode=mode, offset=64)
        base = mm.ctypes.data & ~4095
        end = (mm.ctypes.data + mm.nbytes + 4095) & ~4095
        e = rt.cudaHostRegister(ctypes.c_void_p(base), ctypes.c_size_t(end - base), ctypes.c_uint(flags))
        print(d, mode, flags, e, rt.cudaGetErrorString(e).decode())
        if e == 0:
            rt.cudaHostUnregister(ctypes.c_void_p(base))
        rt.cudaGetLastError()
        del mm
    os.unlink(p)
