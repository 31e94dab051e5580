"""External context numbers on the same box (NOT our kernels): cuBLAS SGEMM
(TF32 off) as the practical FP32 FFMA ceiling, and cuDNN fp32 conv (TF32 off)
on every BASELINE layer.  Prints one JSON object."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402

from paper_2411_15659_b200.workloads import CONFIGS  # noqa: E402


def timeit(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    out = {"sgemm_tflops": {}, "cudnn_fp32": {}}
    for m in (4096, 8192):
        a = torch.randn(m, m, device="cuda")
        b = torch.randn(m, m, device="cuda")
        ms = timeit(lambda: a @ b, 10)
        out["sgemm_tflops"][m] = round(2 * m ** 3 / ms / 1e9, 2)
    for ci, cfg in CONFIGS.items():
        for name, n, g in cfg["layers"]:
            x = torch.randn((n,) + g.input_shape, device="cuda")
            w = torch.randn(g.weights_shape, device="cuda")
            fn = lambda: F.conv2d(x, w, stride=(g.stride_h, g.stride_w),
                                  padding=(g.pad_h, g.pad_w))
            ms = timeit(fn, 10)
            out["cudnn_fp32"][f"cfg{ci}:{name}"] = {"us": round(ms * 1e3, 2),
                                                    "tflops": round(g.flops(n) / ms / 1e9, 2)}
            del x, w
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
