"""Warp-tile 1x1 kernel vs the tile kernels over batch sizes (256 -> 64 @56x56
and 64 -> 64 @56x56): where the warp-tile kernel pays."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from paper_2411_15659_b200 import ConvGeometry, _native, device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from plan_table_sweep import time_plan  # noqa: E402

for ci, hw in ((256, 56), (64, 56), (128, 28), (384, 14)):
    for n in (1, 2, 4, 8, 16, 32, 64):
        g = ConvGeometry(ci, 64, hw, hw, 1, 1)
        x, w = synthetic_layer(g, n, 5)
        xd = torch.from_numpy(x).cuda()
        row = []
        for v in ("1", "0"):
            os.environ["SMMC_1X1_NARROW"] = v
            mod = device.SmmConv2d(g, w, max_batch=n)
            y = mod(xd)
            torch.cuda.synchronize()
            row.append((time_plan(mod, xd, y, 20), time_plan(mod, xd, y, 20, cold=True)))
        print(f"c_i={ci:4d} @{hw} n={n:3d} warp-tile warm {row[0][0]:8.2f} cold {row[0][1]:8.2f} | tiles warm {row[1][0]:8.2f} "
              f"cold {row[1][1]:8.2f} us  ratio cold {row[1][1] / row[0][1]:.2f}", flush=True)
