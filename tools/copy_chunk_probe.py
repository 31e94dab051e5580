"""Chunked H2D/D2H copy-engine behaviour (no compute): per synchronous call,
6 chunks of a 25.7 MB input up and a 25.7 MB output down, with various
stream/event arrangements."""
import time

import torch

MB = 1 << 20
n = 32
xh = torch.empty(n, 64 * 56 * 56).pin_memory()
yh = torch.empty(n, 64 * 56 * 56).pin_memory()
xd = torch.empty_like(xh, device="cuda")
yd = torch.empty_like(yh, device="cuda")
S = [torch.cuda.Stream() for _ in range(6)]
chunks, per = 6, 6


def run(f, reps=10):
    f()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        f()
        torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def sl(c):
    return slice(c * per, min(n, (c + 1) * per))


def h2d_only():
    with torch.cuda.stream(S[0]):
        for c in range(chunks):
            xd[sl(c)].copy_(xh[sl(c)], non_blocking=True)


def h2d_ev():
    with torch.cuda.stream(S[0]):
        for c in range(chunks):
            xd[sl(c)].copy_(xh[sl(c)], non_blocking=True)
            torch.cuda.Event().record(S[0])


def both_indep():
    with torch.cuda.stream(S[0]):
        for c in range(chunks):
            xd[sl(c)].copy_(xh[sl(c)], non_blocking=True)
    with torch.cuda.stream(S[1]):
        for c in range(chunks):
            yh[sl(c)].copy_(yd[sl(c)], non_blocking=True)


def chained(h2d_streams):
    def f():
        evs = []
        for c in range(chunks):
            s = S[c % h2d_streams]
            with torch.cuda.stream(s):
                xd[sl(c)].copy_(xh[sl(c)], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s)
                evs.append(e)
        for c in range(chunks):
            S[5].wait_event(evs[c])
            with torch.cuda.stream(S[5]):
                yh[sl(c)].copy_(yd[sl(c)], non_blocking=True)
    return f


print(f"h2d only         {run(h2d_only):.3f} ms")
print(f"h2d + events     {run(h2d_ev):.3f} ms")
print(f"h2d||d2h indep   {run(both_indep):.3f} ms")
for k in (1, 2, 3):
    print(f"chained d2h(c) after h2d(c), {k} h2d streams  {run(chained(k)):.3f} ms")
