"""Run one BASELINE layer a few times (for ncu / quick timing).

    python tools/prof_layer.py --config 2 --layer conv128@28_n32 [--iters 5] [--mode ffma|exact|bf16_tc|bf16x3_tc]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2411_15659_b200 import device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layer", default="conv128@28_n32")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--mode", default="ffma")
    ap.add_argument("--graph", type=int, default=1)
    a = ap.parse_args()
    for li, (name, n, g) in enumerate(CONFIGS[a.config]["layers"]):
        if name != a.layer:
            continue
        x, w = synthetic_layer(g, n, layer_seed(a.config, li))
        xd = torch.from_numpy(x).cuda()
        if a.mode == "bf16x3_tc":  # fp32-accurate split-bf16: pack + conv every call
            mod = device.Tc3SmmConv2d(g, w)
        elif a.mode == "bf16_tc":  # tcgen05 variant: input packed to bf16 NHWC once
            mod = device.TcSmmConv2d(g, w)
            xd = mod.pack_input(xd)
        else:
            mod = device.SmmConv2d(g, w, mode=a.mode, max_batch=n)
        y = mod(xd)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if a.graph:
            # CUDA graph of `iters` launches: no host launch overhead in the timing
            g_ = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs), torch.cuda.graph(g_, stream=cs):
                for _ in range(a.iters):
                    mod(xd, out=y)
            torch.cuda.synchronize()
            g_.replay()
            torch.cuda.synchronize()
            s.record()
            g_.replay()
            e.record()
        else:
            s.record()
            for _ in range(a.iters):
                mod(xd, out=y)
            e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / a.iters
        print(f"{name}: {ms * 1e3:.1f} us/launch, {g.flops(n) / ms / 1e9:.2f} TFLOP/s")
        return 0
    raise SystemExit(f"no layer {a.layer} in config {a.config}")


if __name__ == "__main__":
    sys.exit(main())
