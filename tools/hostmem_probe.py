"""H2D/D2H bandwidth of pinned host buffers by allocation method (fresh
process each): torch pin_memory (cudaHostAlloc), 4 KB pages + cudaHostRegister,
THP-advised 2 MB-aligned pages + cudaHostRegister."""
import ctypes
import mmap
import subprocess
import sys
import time

import numpy as np
import torch

NB = 64 << 20


def alloc(kind):
    if kind == "pin_memory":
        return torch.empty(NB // 4).pin_memory(), None
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    libc.mmap.restype = ctypes.c_void_p
    libc.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                          ctypes.c_int, ctypes.c_long]
    size = NB + (2 << 20)
    p = libc.mmap(None, size, mmap.PROT_READ | mmap.PROT_WRITE,
                  mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS, -1, 0)
    a = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
    if kind == "thp_register":
        libc.madvise(ctypes.c_void_p(a), ctypes.c_size_t(NB), 14)  # MADV_HUGEPAGE
    arr = np.frombuffer((ctypes.c_char * NB).from_address(a), dtype=np.float32)
    arr[:] = 1.0  # first touch
    t = torch.from_numpy(arr)
    r = torch.cuda.cudart().cudaHostRegister(a, NB, 0)
    assert int(r) == 0, r
    return t, (p, size)


def run(kind):
    h, _ = alloc(kind)
    assert h.is_pinned(), kind
    d = torch.empty(NB // 4, device="cuda")
    d.copy_(h)
    torch.cuda.synchronize()
    res = []
    for direction in ("h2d", "d2h"):
        t = time.perf_counter()
        for _ in range(10):
            if direction == "h2d":
                d.copy_(h, non_blocking=True)
            else:
                h.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        res.append(NB * 10 / (time.perf_counter() - t) / 1e9)
    thp = open("/proc/self/smaps_rollup").read().split("AnonHugePages:")[1].split()[0]
    print(f"{kind:14s} H2D {res[0]:6.1f} GB/s  D2H {res[1]:6.1f} GB/s  (AnonHugePages {thp} kB)",
          flush=True)


if len(sys.argv) > 1:
    run(sys.argv[1])
    sys.exit(0)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
for rep in range(3):
    for kind in ("pin_memory", "register_4k", "thp_register"):
        r = subprocess.run([sys.executable, __file__, kind], capture_output=True, text=True)
        print(r.stdout.strip() or r.stderr[-400:])
