"""Time the tensor-core kernels under forced split-K factors (SMMC_TC_SPLIT)
for chosen BASELINE layers; graph of 20 back-to-back launches per point.

    python tools/tc_split_sweep.py --config 2 --mode bf16x3_tc --splits 1,2,4,8 [--layers a,b]
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15659_b200 import device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402


def graph_us(fn, iters=20):
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(cs), torch.cuda.graph(g, stream=cs):
        for _ in range(iters):
            fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--mode", default="bf16x3_tc")
    ap.add_argument("--splits", default="1,2,4,8")
    ap.add_argument("--layers", default="")
    a = ap.parse_args()
    for li, (name, n, g) in enumerate(CONFIGS[a.config]["layers"]):
        if a.layers and name not in a.layers.split(","):
            continue
        x, w = synthetic_layer(g, n, layer_seed(a.config, li))
        xd = torch.from_numpy(x).cuda()
        res = []
        for sp in a.splits.split(","):
            os.environ["SMMC_TC_SPLIT"] = sp
            if a.mode == "bf16x3_tc":
                mod = device.Tc3SmmConv2d(g, w)
                y = mod(xd)
                us = graph_us(lambda: mod(xd, out=y))
            else:
                mod = device.TcSmmConv2d(g, w)
                xb = mod.pack_input(xd)
                y = mod(xb)
                us = graph_us(lambda: mod(xb, out=y))
            res.append((us, sp))
        os.environ.pop("SMMC_TC_SPLIT", None)
        if a.mode == "bf16x3_tc":
            mod = device.Tc3SmmConv2d(g, w)
            y = mod(xd)
            d = graph_us(lambda: mod(xd, out=y))
        else:
            mod = device.TcSmmConv2d(g, w)
            xb = mod.pack_input(xd)
            y = mod(xb)
            d = graph_us(lambda: mod(xb, out=y))
        print(f"{name:28s} default {d:8.1f} us | " + " ".join(f"S={s}:{u:.1f}" for u, s in res),
              flush=True)


if __name__ == "__main__":
    main()
