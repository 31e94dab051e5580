"""Per-CTA globaltimer timeline of one conv launch (A/B probe build only).

    python -c "from paper_2411_15659_b200 import build; build.build(out='paper_2411_15659_b200/lib/ab/tl.so', defines=['SMMC_PROBE_TL=1'])"
    SMMC_LIB=paper_2411_15659_b200/lib/ab/tl.so python tools/timeline_probe.py --config 2 --layer conv64@56_n1

Stamps per CTA: t0 entry, t1 first stage landed (prologue done), t2 K loop
done, t3 exit.  Printed relative to the earliest entry, in microseconds:
launch ramp (spread of t0), prologue (t1-t0), loop (t2-t1), epilogue /
fixup (t3-t2) and the span (max t3 - min t0).  A 300 MB buffer is written
before the launch so the inputs come from HBM, as in the bench's rotation.
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2411_15659_b200 import _native, device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402


def pct(a, q):
    return float(np.percentile(a, q))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--layer", action="append")
    ap.add_argument("--cold", type=int, default=1)
    a = ap.parse_args()
    lib = _native.lib()
    probe = lib.smmc_probe_timeline
    probe.argtypes = [ctypes.c_void_p, ctypes.c_int]
    flush = torch.empty(300 << 20, dtype=torch.uint8, device="cuda")
    for li, (name, n, g) in enumerate(CONFIGS[a.config]["layers"]):
        if a.layer and name not in a.layer:
            continue
        x, w = synthetic_layer(g, n, layer_seed(a.config, li))
        xd = torch.from_numpy(x).cuda()
        mod = device.SmmConv2d(g, w, max_batch=n)
        y = mod(xd)
        for _ in range(3):
            mod(xd, out=y)
        torch.cuda.synchronize()
        probe(None, 0)
        if a.cold:
            flush.fill_(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        mod(xd, out=y)
        e.record()
        torch.cuda.synchronize()
        buf = np.zeros(16384 * 8, dtype=np.uint64)
        probe(buf.ctypes.data, 16384)
        t = buf.reshape(-1, 8)
        t = t[t[:, 0] != 0].astype(np.int64)
        t0 = t[:, 0].min()
        r = (t[:, :4] - t0) / 1e3
        span = r[:, 3].max()
        sms = len(set(t[:, 4].tolist()))
        print(f"{name}: {len(t)} CTAs on {sms} SMs, event {s.elapsed_time(e) * 1e3:.1f} us, "
              f"CTA span {span:.1f} us")
        # per SM: first and last exit of its CTAs (co-resident CTAs with equal
        # work finishing far apart = unfair issue between CTAs; the SM then
        # runs its last CTA alone)
        by_sm = {}
        for row, sm in zip(r, t[:, 4]):
            by_sm.setdefault(int(sm), []).append(row[3])
        spread = np.array([max(v) - min(v) for v in by_sm.values() if len(v) > 1] or [0.0])
        last = np.array([max(v) for v in by_sm.values()])
        print(f"   per-SM exit spread p50 {pct(spread, 50):.1f} max {spread.max():.1f} us; "
              f"SM done p10 {pct(last, 10):.1f} p50 {pct(last, 50):.1f} max {last.max():.1f} us")
        if (t[:, 7] > 0).all():
            st = (t[:, 7] - t0) / 1e3
            print(f"   setup (entry -> first load issued) p50 {pct(st - r[:, 0], 50):.2f}  "
                  f"loads -> landed p50 {pct(r[:, 1] - st, 50):.2f} us")
        for lab, v in (("entry", r[:, 0]), ("prologue", r[:, 1] - r[:, 0]),
                       ("loop", r[:, 2] - r[:, 1]), ("epilogue", r[:, 3] - r[:, 2]),
                       ("exit", r[:, 3])) + (
                          (("groups", (t[:, 5] - t0) / 1e3 - r[:, 2]),) if (t[:, 5] > 0).all() else ()) + (
                          (("barrier", (t[:, 6] - t[:, 5]) / 1e3), ("reduce", r[:, 3] - (t[:, 6] - t0) / 1e3))
                          if (t[:, 6] > 0).all() else ()):
            print(f"   {lab:9s} min {v.min():7.2f}  p50 {pct(v, 50):7.2f}  p90 {pct(v, 90):7.2f}"
                  f"  max {v.max():7.2f}")


if __name__ == "__main__":
    main()
