"""Forced-plan sweep for the small-batch layers with a correctness check of
every candidate against the CPU oracle (1e-4 * max|ref|) and bitwise
relaunch determinism; per-launch time from a graph of back-to-back launches
(warm) and with an L2-flushing fill before every launch (cold).

    python tools/n1_sweep.py --layers conv64@56_n1,... --cands "4,3,4,5 1,4,3 ..."
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import smm_oracle as orc  # noqa: E402
from paper_2411_15659_b200 import _native, device, repack_weights  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402

sys.path.insert(0, str(Path(__file__).resolve().parent))
from plan_table_sweep import time_plan  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,5")
    ap.add_argument("--layers", required=True)
    ap.add_argument("--cands", required=True, help='space-separated "v,s[,g[,r]]"; ";"-separated per layer')
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    names = a.layers.split(",")
    per_layer = a.cands.split(";")
    for ci in map(int, a.configs.split(",")):
        for li, (name, n, g) in enumerate(CONFIGS[ci]["layers"]):
            if name not in names:
                continue
            cands = (per_layer[names.index(name)] if len(per_layer) > 1 else per_layer[0]).split()
            x, w = synthetic_layer(g, n, layer_seed(ci, li))
            xs = x if n <= 8 else x[:2]
            ref = orc.smm_conv_c(np.ascontiguousarray(xs), repack_weights(w, g), g,
                                 threads=orc.host_threads())
            xd = torch.from_numpy(x).cuda()
            rows = []
            for c in ["default"] + cands:
                os.environ.pop("SMMC_FORCE_PLAN", None)
                if c != "default":
                    os.environ["SMMC_FORCE_PLAN"] = c
                desc = _native.plan_describe(g, n)
                try:
                    mod = device.SmmConv2d(g, w, max_batch=n)
                    y = mod(xd)
                    y2 = mod(xd)
                    torch.cuda.synchronize()
                    err = orc.max_abs_ratio(y[: xs.shape[0]].cpu().numpy(), ref)
                    det = bool(torch.equal(y, y2))
                    warm = time_plan(mod, xd, y, a.iters)
                    cold = time_plan(mod, xd, y, a.iters, cold=True)
                    rows.append((warm, cold, c, err, det, desc))
                except Exception as exc:  # noqa: BLE001
                    print(f"  {name} {c}: FAILED {exc}", flush=True)
            os.environ.pop("SMMC_FORCE_PLAN", None)
            print(f"== {name}", flush=True)
            for warm, cold, c, err, det, desc in sorted(rows):
                ok = "ok" if err <= 1e-4 and det else "BAD"
                print(f"  {c:12s} warm {warm:7.2f} us cold {cold:7.2f} us  err {err:.1e} det {det} {ok}  {desc[6:120]}",
                      flush=True)


if __name__ == "__main__":
    main()
