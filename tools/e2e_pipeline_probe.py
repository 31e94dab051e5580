"""Chunked H2D/conv/D2H pipeline built from torch streams around the device
entry, to compare against smmc_conv2d_fwd_f32_host (diagnostic)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15659_b200 import device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402

name, n, g = CONFIGS[2]["layers"][4]
x, w = synthetic_layer(g, n, layer_seed(2, 4))
xh = torch.from_numpy(x).pin_memory()
yh = torch.empty((n,) + g.output_shape).pin_memory()
xd = torch.empty_like(xh, device="cuda")
yd = torch.empty_like(yh, device="cuda")
mod = device.SmmConv2d(g, w, max_batch=n)
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
for chunks in (1, 2, 4, 8):
    per = n // chunks

    def run():
        evs = []
        for c in range(chunks):
            sl = slice(c * per, (c + 1) * per)
            with torch.cuda.stream(s_in):
                xd[sl].copy_(xh[sl], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_in)
            s_c.wait_event(e)
            with torch.cuda.stream(s_c):
                mod(xd[sl], out=yd[sl])
                e2 = torch.cuda.Event()
                e2.record(s_c)
            s_out.wait_event(e2)
            with torch.cuda.stream(s_out):
                yh[sl].copy_(yd[sl], non_blocking=True)
        s_out.synchronize()

    run()
    t = time.perf_counter()
    for _ in range(5):
        run()
    dt = (time.perf_counter() - t) / 5
    print(f"{name} chunks={chunks}: {dt * 1e3:.3f} ms")
