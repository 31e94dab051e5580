"""Per-layer timing of the host-buffer entry (smmc_conv2d_fwd_f32_host) vs the
pure transfer time, for BASELINE config C."""
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

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
lib = _native.lib()
for li, (name, n, g) in enumerate(CONFIGS[cfg]["layers"]):
    x, w = synthetic_layer(g, n, layer_seed(cfg, li))
    ws = np.ascontiguousarray(w.transpose(1, 3, 2, 0))
    xh = torch.from_numpy(_native.pinned_copy(x))
    wh = torch.from_numpy(_native.pinned_copy(ws))
    yh = torch.from_numpy(_native.pinned_empty((n,) + g.output_shape))
    G = _native.Geom.of(g, n)

    def call():
        _native.check(lib.smmc_conv2d_fwd_f32_host(
            ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(wh.data_ptr()),
            ctypes.c_void_p(yh.data_ptr()), ctypes.byref(G), 0, 0), "e2e")

    call()
    t = time.perf_counter()
    for _ in range(5):
        call()
    dt = (time.perf_counter() - t) / 5
    h2d = (xh.numel() + wh.numel()) * 4
    d2h = yh.numel() * 4
    print(f"{name:28s} {dt * 1e3:8.3f} ms  h2d {h2d / 1e6:7.1f} MB d2h {d2h / 1e6:7.1f} MB  "
          f"serial-copy bound {(h2d + d2h) / 55e9 * 1e3:6.3f} ms  overlap bound "
          f"{max(h2d, d2h) / 55e9 * 1e3:6.3f} ms  {g.flops(n) / dt / 1e12:6.2f} TF")

# the bench's access pattern: every layer once per step, steps back to back
calls = []
for li, (name, n, g) in enumerate(CONFIGS[cfg]["layers"]):
    x, w = synthetic_layer(g, n, layer_seed(cfg, li))
    ws = np.ascontiguousarray(w.transpose(1, 3, 2, 0))
    xh = torch.from_numpy(_native.pinned_copy(x))
    wh = torch.from_numpy(_native.pinned_copy(ws))
    yh = torch.from_numpy(_native.pinned_empty((n,) + g.output_shape))
    calls.append((xh, wh, yh, _native.Geom.of(g, n), g.flops(n)))


def step():
    for xh, wh, yh, G, _ in calls:
        _native.check(lib.smmc_conv2d_fwd_f32_host(
            ctypes.c_void_p(xh.data_ptr()), ctypes.c_void_p(wh.data_ptr()),
            ctypes.c_void_p(yh.data_ptr()), ctypes.byref(G), 0, 0), "e2e")


step()
t = time.perf_counter()
for _ in range(5):
    step()
dt = (time.perf_counter() - t) / 5
print(f"step: {dt * 1e3:.3f} ms, {sum(c[4] for c in calls) / dt / 1e12:.2f} TF")
