"""Repeat host-entry and device-path launches of the N=1 / weight-heavy
layers and compare every result bitwise with the first (intermittent-failure
hunt; compute-sanitizer is unavailable on the pool)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, _native, device
from paper_2411_15659_b200.tensors import synthetic_layer
from oracle import smm_oracle as orc
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cases = [((256, 200, 7, 7, 3, 3, 1, 1, 1, 1), 2), ((512, 512, 7, 7, 3, 3, 1, 1, 1, 1), 1),
         ((128, 96, 5, 6, 5, 3, 1, 2, 2, 1), 3), ((64, 70, 4, 4, 1, 1, 1, 1, 0, 0), 1),
         ((64, 64, 56, 56, 3, 3, 1, 1, 1, 1), 1), ((128, 128, 28, 28, 3, 3, 1, 1, 1, 1), 1),
         ((256, 256, 14, 14, 3, 3, 1, 1, 1, 1), 1)]
bad = 0
for gt, n in cases:
    g = ConvGeometry(*gt)
    x, w = synthetic_layer(g, n, 31)
    ws = smm.repack_weights(w, g)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    xd = torch.from_numpy(x).cuda(); wd = torch.from_numpy(ws).cuda()
    first = None
    nbad = {"host": 0, "hostpin": 0, "dev": 0}
    for r in range(reps):
        for kind in ("host", "hostpin", "dev"):
            if kind == "host":
                y = smm.smm_conv_batched(x, ws, g)
            elif kind == "hostpin":
                y = smm.smm_conv_batched(_native.pinned_copy(x), _native.pinned_copy(ws), g)
            else:
                y = device.conv2d(xd, wd, g).cpu().numpy()
            if first is None:
                first = y.copy()
                print(gt, n, "first err", orc.max_abs_ratio(y, ref), _native.plan_describe(g, n), flush=True)
            if not np.array_equal(y, first):
                nbad[kind] += 1
                if nbad[kind] <= 3:
                    d = np.abs(y - first)
                    idx = np.argwhere(d > 0)
                    print("  MISMATCH", kind, r, "err", orc.max_abs_ratio(y, ref), "n_diff", len(idx),
                          "first idx", idx[:4].tolist(), flush=True)
    print(gt, n, "mismatches", nbad, flush=True)
    bad += sum(nbad.values())
print("TOTAL_BAD", bad)
