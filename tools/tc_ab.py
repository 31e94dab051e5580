"""Time the bf16 tensor-core conv on BASELINE layers (graph replay), for A/B
of SMMC_TC_KERNEL=box|halo.  python tools/tc_ab.py cfg:layer ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2411_15659_b200 import device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402

for item in sys.argv[1:]:
    c, name = item.split(":")
    for li, (nm, n, g) in enumerate(CONFIGS[int(c)]["layers"]):
        if nm != name:
            continue
        x, w = synthetic_layer(g, n, layer_seed(int(c), li))
        mod = device.TcSmmConv2d(g, w)
        xb = mod.pack_input(torch.from_numpy(x).cuda())
        y = mod(xb)
        gr = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        it = 20
        with torch.cuda.stream(cs), torch.cuda.graph(gr, stream=cs):
            for _ in range(it):
                mod(xb, out=y)
        torch.cuda.synchronize()
        gr.replay()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        gr.replay()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / it * 1e3
        print(f"{nm:28s} {us:8.1f} us {g.flops(n) / us / 1e6:8.1f} TF", flush=True)
