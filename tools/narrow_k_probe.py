"""Fixed cost vs per-channel-block cost of the warp-tile 1x1 kernel:
time (c_i -> 64 @56x56, N=8) for several c_i (graph of back-to-back launches)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from paper_2411_15659_b200 import ConvGeometry, _native, device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from plan_table_sweep import time_plan  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
for ci in (64, 128, 192, 256, 320, 384):
    g = ConvGeometry(ci, 64, 56, 56, 1, 1)
    x, w = synthetic_layer(g, n, 5)
    xd = torch.from_numpy(x).cuda()
    mod = device.SmmConv2d(g, w, max_batch=n)
    y = mod(xd)
    torch.cuda.synchronize()
    warm = time_plan(mod, xd, y, 20)
    cold = time_plan(mod, xd, y, 20, cold=True)
    fl = 2.0 * n * 64 * 56 * 56 * ci
    print(f"c_i={ci:4d} n={n} warm {warm:7.2f} us cold {cold:7.2f} us  {fl / warm / 1e6:6.1f} TFLOP/s warm  "
          f"{_native.plan_describe(g, n)[-60:]}", flush=True)
