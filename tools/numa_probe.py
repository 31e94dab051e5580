"""Pinned-host H2D/D2H bandwidth vs the process's CPU/NUMA placement.
python tools/numa_probe.py  (prints topology, then GB/s per placement)"""
import os
import subprocess
import sys
import time

import torch


def bw(nbytes=64 << 20, reps=10):
    h = torch.empty(nbytes // 4).pin_memory()
    d = torch.empty_like(h, device="cuda")
    d.copy_(h)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    up = nbytes * reps / (time.perf_counter() - t) / 1e9
    t = time.perf_counter()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    down = nbytes * reps / (time.perf_counter() - t) / 1e9
    return up, down


if len(sys.argv) > 1 and sys.argv[1] == "child":
    up, down = bw()
    print(f"  cpus {sys.argv[2]:>12s}: H2D {up:6.1f} GB/s  D2H {down:6.1f} GB/s", flush=True)
    sys.exit(0)

print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print(subprocess.run(["lscpu"], capture_output=True, text=True).stdout)
nodes = sorted(os.listdir("/sys/devices/system/node")) if os.path.isdir("/sys/devices/system/node") else []
placements = [("all", None)]
for nd in nodes:
    if nd.startswith("node"):
        with open(f"/sys/devices/system/node/{nd}/cpulist") as f:
            placements.append((nd, f.read().strip()))
try:
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    mask = pynvml.nvmlDeviceGetCpuAffinity(hnd, 4)
    cpus = [i for w, m in enumerate(mask) for i in range(64) if (m >> i) & 1 for i in [w * 64 + i]]
    print("NVML GPU0 cpu affinity:", cpus[:8], "...", len(cpus), "cpus")
except Exception as e:  # noqa: BLE001
    print("nvml:", e)
for name, cpulist in placements:
    cmd = [sys.executable, __file__, "child", cpulist or "all"]
    if cpulist:
        cmd = ["taskset", "-c", cpulist] + cmd
    print(name, end="")
    r = subprocess.run(cmd, capture_output=True, text=True)
    print(r.stdout or r.stderr[-300:])
