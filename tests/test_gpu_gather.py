"""GPU parity of the fused output-channel-shard conv + all-gather
(smmc_conv2d_fwd_f32_gather).

One GPU is available, so P ranks are emulated one after another in this
process (no rank waits on another): rank r convolves its channel slice and
its placement pass stores the result into all P replica buffers — exactly
what it does with NVLink-mapped peer buffers.  Afterwards every replica must
hold the full output (oracle tolerance) and the replicas must be bitwise
identical."""

import numpy as np
import pytest

from oracle import smm_oracle as orc
from paper_2411_15659_b200 import ConvGeometry, DeviceError, ShapeMismatchError, _native
from paper_2411_15659_b200.parallel import cout_geometry, cout_shard
from paper_2411_15659_b200.tensors import synthetic_layer
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _emulate(g, n, world, seed):
    import torch
    from paper_2411_15659_b200 import device
    x, w = synthetic_layer(g, n, seed)
    ws = np.ascontiguousarray(w.transpose(1, 3, 2, 0))
    xd = torch.from_numpy(x).cuda()
    outs = [torch.full((n,) + g.output_shape, float("nan"), device="cuda") for _ in range(world)]
    for r in range(world):
        lo, hi = cout_shard(g.out_channels, r, world)
        if hi == lo:
            continue
        wd = torch.from_numpy(np.ascontiguousarray(ws[..., lo:hi])).cuda()
        device.conv2d_gather(xd, wd, outs, cout_geometry(g, lo, hi), lo, g.out_channels)
    torch.cuda.synchronize()
    return x, w, [o.cpu().numpy() for o in outs]


CASES = [
    ("cfg5_512@7_n8", CONFIGS[5]["layers"][3][2], 8, layer_seed(5, 3)),
    ("odd", ConvGeometry(24, 37, 11, 9, 3, 3, pad_h=1, pad_w=1), 3, 4),
    ("1x1", ConvGeometry(32, 64, 8, 8, 1, 1), 2, 6),
]


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("name,g,n,seed", CASES, ids=[c[0] for c in CASES])
def test_gather_emulated_ranks(name, g, n, seed, world):
    x, w, outs = _emulate(g, n, world, seed)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    for o in outs:
        assert np.isfinite(o).all()
        assert orc.max_abs_ratio(o, ref) <= TOL
        assert np.array_equal(o, outs[0])


@pytest.mark.parametrize("force", ["3,0", "1,8", "0,1", "2,3"])
def test_gather_every_plan_kind(monkeypatch, force):
    """Stream-K, split-K and plain plans are all recast to the placement pass."""
    monkeypatch.setenv("SMMC_FORCE_PLAN", force)
    g = ConvGeometry(64, 96, 14, 14, 3, 3, pad_h=1, pad_w=1)
    x, w, outs = _emulate(g, 4, 3, 12)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    for o in outs:
        assert orc.max_abs_ratio(o, ref) <= TOL


def test_gather_argument_errors():
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(8, 16, 6, 6, 3, 3, pad_h=1, pad_w=1)
    gl = cout_geometry(g, 0, 8)
    x = torch.zeros((2,) + g.input_shape, device="cuda")
    w = torch.zeros(gl.weights_smm_shape, device="cuda")
    out = torch.zeros((2,) + g.output_shape, device="cuda")
    with pytest.raises(ShapeMismatchError):
        device.conv2d_gather(x, w, [], gl, 0, 16)
    with pytest.raises(ShapeMismatchError):
        device.conv2d_gather(x, w, [out] * 9, gl, 0, 16)
    with pytest.raises(ShapeMismatchError):        # window [10, 18) outside 16 channels
        device.conv2d_gather(x, w, [out], gl, 10, 16)
    with pytest.raises(ShapeMismatchError):        # misaligned raw replica address
        device.conv2d_gather(x, w, [out, out.data_ptr() + 4], gl, 0, 16)


def test_ipc_handles():
    import torch
    t = torch.empty(4096, device="cuda")
    h0, o0 = _native.ipc_handle(t.data_ptr())
    h1, o1 = _native.ipc_handle(t[256:].data_ptr())
    assert h0 == h1 and o1 - o0 == 1024 and len(h0) == _native.SMMC_IPC_HANDLE_BYTES
    with pytest.raises(DeviceError):               # CUDA refuses to map its own process
        _native.ipc_open(h0, o0)
    # a reported CUDA failure must not leak into the next launch's status
    from paper_2411_15659_b200 import device
    g = ConvGeometry(8, 8, 6, 6, 3, 3, pad_h=1, pad_w=1)
    y = device.conv2d(torch.zeros((1,) + g.input_shape, device="cuda"),
                      torch.zeros(g.weights_smm_shape, device="cuda"), g, mode="exact")
    torch.cuda.synchronize()
    assert float(y.abs().max()) == 0.0
