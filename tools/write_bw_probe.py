"""HBM bandwidth of write-dominated traffic (the bf16 1x1 layer's shape:
103 MB read + 822 MB written): fill, copy, and strided-channel writes."""
import torch

n = 822 * 1024 * 1024 // 4
y = torch.empty(n, device="cuda")
x = torch.empty(103 * 1024 * 1024 // 2, dtype=torch.bfloat16, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (("fill 822 MB", lambda: y.fill_(1.0), 4 * n),
                         ("copy 411+411 MB", lambda: y[n // 2:].copy_(y[:n // 2]), 4 * n),
                         ("read 103 MB bf16 + fill 822 MB", lambda: (x.sum(), y.fill_(2.0)),
                          4 * n + 2 * x.numel())):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{name:34s} {ms * 1e3:8.1f} us  {nbytes / ms / 1e9:7.1f} GB/s")
