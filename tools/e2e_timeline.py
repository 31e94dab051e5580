"""CUPTI timeline (torch.profiler) of one host-entry call: when each H2D,
kernel and D2H ran.  python tools/e2e_timeline.py cfg layer"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2411_15659_b200 import _native  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402

cfg, lname = int(sys.argv[1]), sys.argv[2]
li, (name, n, g) = next((i, l) for i, l in enumerate(CONFIGS[cfg]["layers"]) if l[0] == lname)
x, w = synthetic_layer(g, n, layer_seed(cfg, li))
# page-locked via the library's allocator (cudaHostRegister'd pages, 55 GB/s
# H2D here; torch's pin_memory buffers run ~33)
xh = torch.from_numpy(_native.pinned_copy(x))
wh = torch.from_numpy(_native.pinned_copy(np.ascontiguousarray(w.transpose(1, 3, 2, 0))))
yh = torch.from_numpy(_native.pinned_empty((n,) + g.output_shape))
lib = _native.lib()
G = _native.Geom.of(g, n)


def host():
    _native.check(lib.smmc_conv2d_fwd_f32_host(
        ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(wh.data_ptr()),
        ctypes.c_void_p(yh.data_ptr()), ctypes.byref(G), 0, 0), "e2e")


for _ in range(3):
    host()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    host()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
for e in evs:
    print(f"{e.time_range.start - t0:9.1f} us {e.time_range.elapsed_us():8.1f} us  {e.name[:70]}")

if len(sys.argv) > 3:  # torch-stream replica of the same chunk pipeline, for comparison
    from paper_2411_15659_b200 import device
    chunks = int(sys.argv[3])
    xd, wd = torch.empty_like(xh, device="cuda"), torch.empty_like(wh, device="cuda")
    yd = torch.empty_like(yh, device="cuda")
    s1, s2, sc = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    per = (n + chunks - 1) // chunks

    def pipe():
        with torch.cuda.stream(s1):
            wd.copy_(wh, non_blocking=True)
        for c in range(chunks):
            a, b = c * per, min(n, (c + 1) * per)
            if a >= b:
                break
            e1, e2 = torch.cuda.Event(), torch.cuda.Event()
            with torch.cuda.stream(s1):
                xd[a:b].copy_(xh[a:b], non_blocking=True)
                e1.record(s1)
            with torch.cuda.stream(sc):
                sc.wait_event(e1)
                device.conv2d(xd[a:b], wd, g, out=yd[a:b])
                e2.record(sc)
            with torch.cuda.stream(s2):
                s2.wait_event(e2)
                yh[a:b].copy_(yd[a:b], non_blocking=True)
        torch.cuda.synchronize()

    for _ in range(3):
        pipe()
    import time
    t = time.perf_counter()
    for _ in range(10):
        pipe()
    print(f"py pipe {chunks} chunks: {(time.perf_counter() - t) / 10 * 1e3:.3f} ms per synchronous call")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        pipe()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    t0 = evs[0].time_range.start if evs else 0
    for e in evs:
        print(f"{e.time_range.start - t0:9.1f} us {e.time_range.elapsed_us():8.1f} us  {e.name[:70]}")
