"""Does the host entry overlap H2D / D2H?  Times, for one layer: pure H2D,
pure D2H, both concurrently (torch copies on two streams), and the host
entry smmc_conv2d_fwd_f32_host.  python tools/e2e_overlap_probe.py cfg layer"""
import ctypes
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15659_b200 import _native  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402

cfg, lname = int(sys.argv[1]), sys.argv[2]
li, (name, n, g) = next((i, l) for i, l in enumerate(CONFIGS[cfg]["layers"]) if l[0] == lname)
x, w = synthetic_layer(g, n, layer_seed(cfg, li))
ws = np.ascontiguousarray(w.transpose(1, 3, 2, 0))
xh = torch.from_numpy(x).pin_memory()
wh = torch.from_numpy(ws).pin_memory()
yh = torch.empty((n,) + g.output_shape).pin_memory()
xd, wd, yd = xh.cuda(), wh.cuda(), torch.empty_like(yh, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
print("pinned:", xh.is_pinned(), wh.is_pinned(), yh.is_pinned())


def timeit(f, reps=10):
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def h2d():
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
        wd.copy_(wh, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        yh.copy_(yd, non_blocking=True)


def both():
    h2d()
    d2h()


lib = _native.lib()
G = _native.Geom.of(g, n)


def host():
    _native.check(lib.smmc_conv2d_fwd_f32_host(
        ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(wh.data_ptr()),
        ctypes.c_void_p(yh.data_ptr()), ctypes.byref(G), 0, 0), "e2e")


hb = (xh.numel() + wh.numel()) * 4
db = yh.numel() * 4
for nm, f, b in (("h2d", h2d, hb), ("d2h", d2h, db), ("both", both, hb + db), ("host entry", host, hb + db)):
    ms = timeit(f)
    print(f"{name} {nm:10s} {ms:7.3f} ms  {b / ms / 1e6:6.1f} GB/s")

# Python replica of the host entry's chunk pipeline (torch streams + device conv)
from paper_2411_15659_b200 import device  # noqa: E402

sc = torch.cuda.Stream()
wsd = torch.zeros(max(1, _native.workspace_bytes(g, n)), dtype=torch.uint8, device="cuda")
for chunks in (1, 2, 4, 8, 16):
    if chunks > n:
        break
    per = (n + chunks - 1) // chunks
    ev_in = [torch.cuda.Event() for _ in range(chunks)]
    ev_c = [torch.cuda.Event() for _ in range(chunks)]

    def pipe():
        with torch.cuda.stream(s1):
            wd.copy_(wh, non_blocking=True)
        for c in range(chunks):
            a, b = c * per, min(n, (c + 1) * per)
            if a >= b:
                break
            with torch.cuda.stream(s1):
                xd[a:b].copy_(xh[a:b], non_blocking=True)
                ev_in[c].record(s1)
            with torch.cuda.stream(sc):
                sc.wait_event(ev_in[c])
                device.conv2d(xd[a:b], wd, g, out=yd[a:b])
                ev_c[c].record(sc)
            with torch.cuda.stream(s2):
                s2.wait_event(ev_c[c])
                yh[a:b].copy_(yd[a:b], non_blocking=True)

    ms = timeit(pipe)
    print(f"{name} py-pipe chunks={chunks:2d} {ms:7.3f} ms")
