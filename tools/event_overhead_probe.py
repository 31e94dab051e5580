"""Does the bench's per-layer event recording inside the timed graph cost
time?  Config-2 step as a graph with and without external per-layer events
(same rotating replicas as bench.py)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_15659_b200 import _native, device  # noqa: E402
from paper_2411_15659_b200.tensors import synthetic_layer  # noqa: E402
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
R, STEPS = 5, 10
layers = []
for li, (name, n, g) in enumerate(CONFIGS[cfg]["layers"]):
    x, w = synthetic_layer(g, n, layer_seed(cfg, li))
    ws = np.ascontiguousarray(w.transpose(1, 3, 2, 0))
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(ws).cuda()
    layers.append(dict(g=g, x=[xd.clone() for _ in range(R)], w=[wd.clone() for _ in range(R)],
                       y=[torch.empty((n,) + g.output_shape, device="cuda") for _ in range(R)],
                       ws=torch.zeros(max(_native.workspace_bytes(g, n), 16), dtype=torch.uint8,
                                      device="cuda")))


def step(r, evs=None):
    for li, L in enumerate(layers):
        device.conv2d(L["x"][r], L["w"][r], L["g"], out=L["y"][r], workspace=L["ws"])
        if evs is not None:
            evs[li].record()


def capture(with_events, kind):
    evs = [[torch.cuda.Event(enable_timing=True, external=(kind == "external"))
            for _ in layers] for _ in range(STEPS)]
    g_ = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cs), torch.cuda.graph(g_, stream=cs):
        for s in range(STEPS):
            step(s % R, evs[s] if with_events else None)
    torch.cuda.synchronize()
    return g_


for _ in range(3):
    step(0)
torch.cuda.synchronize()
for name, we, kind in [("no events", False, None), ("external events", True, "external")] * 4:
    g_ = capture(we, kind)
    g_.replay()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g_.replay()
    e.record()
    torch.cuda.synchronize()
    print(f"{name:16s} {s.elapsed_time(e) / STEPS * 1e3:8.1f} us per step", flush=True)

