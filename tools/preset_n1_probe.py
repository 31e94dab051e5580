"""Per-layer kernel time (CUDA graph of back-to-back launches) of the preset
networks at the reference harness's batch of 1, with the chosen plan.
    python tools/preset_n1_probe.py [--net vgg16] [--batch 1] [--force "v,s,g,r"]"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15659_b200 import _native, device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import network_geometries  # noqa: E402


def time_layer(g, n, iters):
    x, w = synthetic_layer(g, n, 1)
    xd = torch.from_numpy(x).cuda()
    mod = device.SmmConv2d(g, w, max_batch=n)
    y = mod(xd)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs), torch.cuda.graph(gr, stream=cs):
        for _ in range(iters):
            mod(xd, out=y)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    gr.replay()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--net", default="vgg16")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cands", default="", help='space-separated forced plans "v,s[,g[,r]]" tried per layer')
    ap.add_argument("--sweep", default="", help="one of the paper's sweeps instead of a network")
    ap.add_argument("--auto", action="store_true")
    ap.add_argument("--autotune", action="store_true", help="default vs smmc_autotune_f32 per layer")
    ap.add_argument("--quiet", action="store_true")
    a = ap.parse_args()
    seen = set()
    total = [0.0, 0.0]
    if a.sweep:
        from paper_2411_15659_b200.harness import sweep
        layers = [(sp.name, sp.geometry) for sp in sweep(a.sweep)]
    else:
        layers = network_geometries(a.net)
    for name, g in layers:
        key = (g.in_channels, g.out_channels, g.in_h, g.in_w, g.k_h, g.stride_h)
        if key in seen:
            continue
        seen.add(key)
        fl = 2.0 * a.batch * g.out_channels * g.out_h * g.out_w * g.in_channels * g.k_h * g.k_w
        os.environ.pop("SMMC_FORCE_PLAN", None)
        _native.autotune_clear()
        us = time_layer(g, a.batch, a.iters)
        if a.autotune:
            rep = _native.autotune(g, a.batch)
            ut = time_layer(g, a.batch, a.iters)
            print(f"{name:10s} default {us:7.1f} us -> tuned {ut:7.1f} us ({us / ut:4.2f}x)  [{rep}]", flush=True)
            total[0] += us
            total[1] += ut
            continue
        print(f"{name:10s} {g.in_channels:4d}->{g.out_channels:4d} @{g.in_h:3d} k{g.k_h} s{g.stride_h}: "
              f"{us:8.1f} us {fl / us / 1e6:6.2f} TF {100 * fl / us / 1e6 / 74.45:5.1f}%  "
              f"{_native.plan_describe(g, a.batch)[:110]}", flush=True)
        cands = a.cands.split()
        if a.auto:  # in-kernel split plans sized to ~0.5, 1, 2 CTAs per SM
            m = a.batch * g.out_h * g.out_w
            kt = g.k_h * g.k_w * (g.in_channels // 16) if g.in_channels % 16 == 0 else 0
            for v, bm, bn, gs in ((3, 64, 128, (2,)), (4, 64, 64, (2, 4)), (1, 128, 64, (2, 4))):
                tiles = -(-m // bm) * -(-g.out_channels // bn)
                for target in (74, 111, 148, 222, 296):
                    sp = target // tiles
                    for gg in gs:
                        if 2 <= sp <= 32 and kt and kt // sp >= gg:
                            c = f"{v},{sp},{gg},5"
                            if c not in cands:
                                cands.append(c)
            cands += ["3,0", "1,0"]
        best = (us, "default")
        for c in cands:
            os.environ["SMMC_FORCE_PLAN"] = c
            try:
                u2 = time_layer(g, a.batch, a.iters)
                best = min(best, (u2, c))
                if not a.quiet:
                    print(f"      {c:10s} {u2:8.1f} us  {_native.plan_describe(g, a.batch)[:100]}", flush=True)
            except Exception as ex:  # noqa: BLE001
                if not a.quiet:
                    print(f"      {c:10s} failed: {str(ex)[:80]}", flush=True)
        os.environ.pop("SMMC_FORCE_PLAN", None)
        if cands:
            print(f"      best {best[1]:12s} {best[0]:8.1f} us ({us / best[0]:.2f}x default)", flush=True)
    if a.autotune:
        print(f"{a.sweep or a.net} distinct conv layers at batch {a.batch}: default {total[0]:.1f} us -> tuned {total[1]:.1f} us")


if __name__ == "__main__":
    main()
