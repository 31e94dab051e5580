"""Sweep forced FFMA plans for every BASELINE layer (one process), print the
best plan per layer as a table (for the per-shape tuning table in conv_ffma.cu).

    python tools/plan_table_sweep.py [--configs 2,3,5] > sweep.txt
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15659_b200 import _native, device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402


_FLUSH = None


def _flush_buf():
    global _FLUSH
    if _FLUSH is None:  # 2x the 126 MB L2
        _FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    return _FLUSH


def time_plan(mod, xd, y, iters, cold=False):
    """Per-launch time (us) from one graph replay of `iters` launches; cold:
    an L2-flushing 256 MB fill before every launch, its own time subtracted."""
    if cold:
        fb = _flush_buf()
        g_f = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs), torch.cuda.graph(g_f, stream=cs):
            for _ in range(iters):
                fb.fill_(1)
        torch.cuda.synchronize()
        g_f.replay()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        g_f.replay()
        e.record()
        torch.cuda.synchronize()
        flush_ms = s.elapsed_time(e)
    g_ = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs), torch.cuda.graph(g_, stream=cs):
        for _ in range(iters):
            if cold:
                fb.fill_(1)
            mod(xd, out=y)
    torch.cuda.synchronize()
    g_.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g_.replay()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) - (flush_ms if cold else 0.0)
    return ms / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,5,4")
    ap.add_argument("--cold", action="store_true", help="flush L2 before every launch")
    ap.add_argument("--max-gflop", type=float, default=1e9, help="skip larger layers")
    ap.add_argument("--layers", default="", help="comma-separated layer names (default: all)")
    ap.add_argument("--cands", default="", help='forced plans "v,s v,s ..." (default: the grid)')
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    out = {}
    seen = set()
    for ci in map(int, a.configs.split(",")):
        for li, (name, n, g) in enumerate(CONFIGS[ci]["layers"]):
            key = (n,) + g.as_abi(n)[1:]
            if key in seen:
                continue
            seen.add(key)
            if g.flops(n) > a.max_gflop * 1e9:
                continue
            if a.layers and name not in a.layers.split(","):
                continue
            x, w = synthetic_layer(g, n, layer_seed(ci, li))
            xd = torch.from_numpy(x).cuda()
            small = g.flops(n) < 2e9
            cands = ([(v, s) for v in (0, 1, 3) for s in (4, 8, 16, 24, 32, 0)] if small else
                     [(v, s) for v in (0, 1, 2, 3) for s in (1, 2, 3, 4, 0)])
            if a.cands:
                cands = [tuple(map(int, c.split(","))) for c in a.cands.split()]
            iters = 20 if g.flops(n) < 20e9 else 3
            res = []
            os.environ.pop("SMMC_FORCE_PLAN", None)
            mod = device.SmmConv2d(g, w)
            y = mod(xd)
            default = (time_plan(mod, xd, y, iters, a.cold), _native.plan_describe(g, n))
            for c in cands:
                v, s = c[0], ",".join(map(str, c[1:]))
                os.environ["SMMC_FORCE_PLAN"] = f"{v},{s}"
                mod = device.SmmConv2d(g, w)
                y = mod(xd)
                try:
                    res.append((time_plan(mod, xd, y, iters, a.cold), v, s))
                except Exception as exc:  # noqa: BLE001
                    print(f"  {name} {v},{s}: {exc}", file=sys.stderr)
            os.environ.pop("SMMC_FORCE_PLAN", None)
            res.sort()
            best = res[0]
            nxt = " ".join(f"{r[0]:.1f} ({r[1]},{r[2]})" for r in res[1:4])
            print(f"{name:32s} default {default[0]:9.1f} us | best {best[0]:9.1f} us plan {best[1]},{best[2]}"
                  f" | next {nxt}", flush=True)
            out[name] = {"key": key, "default_us": default[0], "default_plan": default[1],
                         "best": [best[1], best[2]], "best_us": best[0],
                         "all": [[r[1], r[2], round(r[0], 2)] for r in res]}
            del xd, mod, y
            torch.cuda.empty_cache()
    Path(a.out or "gpurun_out/plan_sweep%s.json" % ("_cold" if a.cold else "")).write_text(
        json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
