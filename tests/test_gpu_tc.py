"""GPU parity of the separately labelled bf16 tensor-core variant (tcgen05):
max|y - ref| <= 2e-2 * max|ref| against the fp32 oracle (BASELINE config 5)."""

import numpy as np
import pytest

from oracle import smm_oracle as orc
from paper_2411_15659_b200 import BackendUnsupportedError, ConvGeometry
from paper_2411_15659_b200.tensors import synthetic_layer
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed

pytestmark = pytest.mark.gpu

TOL_BF16 = 2e-2


def _run_tc(g, n, seed):
    import torch
    from paper_2411_15659_b200 import device
    x, w = synthetic_layer(g, n, seed)
    layer = device.TcSmmConv2d(g, w)
    xd = torch.from_numpy(x).cuda()
    y = layer(layer.pack_input(xd))
    torch.cuda.synchronize()
    return x, w, y.cpu().numpy()


SMALL = [
    (64, 64, 14, 14, 3, 3, 1, 1, 1, 1, 2),
    (64, 128, 28, 28, 3, 3, 1, 1, 1, 1, 1),
    (128, 64, 7, 7, 3, 3, 1, 1, 1, 1, 3),
    (96, 256, 27, 27, 5, 5, 1, 1, 2, 2, 1),
    (64, 256, 12, 12, 1, 1, 1, 1, 0, 0, 3),
    (256, 64, 56, 56, 1, 1, 1, 1, 0, 0, 1),
    (32, 40, 9, 11, 3, 3, 1, 1, 1, 1, 2),
    (8, 130, 6, 5, 3, 5, 1, 1, 1, 2, 2),
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: "x".join(map(str, c)))
def test_tc_small_shapes(case):
    *gt, n = case
    g = ConvGeometry(*gt)
    x, w, y = _run_tc(g, n, 11)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    err = orc.max_abs_ratio(y, ref)
    assert err <= TOL_BF16, err
    assert err >= 1e-5  # it really is bf16 (not a silent fp32 path)


TC_LAYERS = [(5, li, name, n, g) for li, (name, n, g) in enumerate(CONFIGS[5]["layers"])]


@pytest.mark.parametrize("ci,li,name,n,g", TC_LAYERS, ids=[l[2] for l in TC_LAYERS])
def test_tc_config5_full_size(ci, li, name, n, g):
    x, w, y = _run_tc(g, n, layer_seed(ci, li))
    assert np.isfinite(y).all()
    samples = [0, n - 1]
    ref = orc.smm_conv_c(np.ascontiguousarray(x[samples]), orc.repack(w), g,
                         threads=orc.host_threads())
    assert orc.max_abs_ratio(y[samples], ref) <= TOL_BF16


def test_tc_rejects_strided():
    from paper_2411_15659_b200 import device
    g = ConvGeometry(16, 16, 16, 16, 3, 3, stride_h=2, stride_w=2, pad_h=1, pad_w=1)
    assert not device.tc_supported(g)
    with pytest.raises(BackendUnsupportedError):
        device.TcSmmConv2d(g, np.zeros(g.weights_shape, np.float32))


@pytest.mark.parametrize("bn", ["128", "128p", "128p2", "256"])
@pytest.mark.parametrize("case", [
    (64, 512, 14, 14, 3, 3, 1, 1, 1, 1, 3),   # two N=256 tiles, ragged last M tile
    (32, 320, 9, 11, 3, 3, 1, 1, 1, 1, 2),    # c_o % 256 != 0: partial second N tile
    (128, 256, 20, 20, 3, 3, 1, 1, 1, 1, 40),  # > 2 tiles per persistent CTA
    (64, 256, 8, 12, 1, 1, 1, 1, 0, 0, 5),     # 1x1 at N=256: tiles straddle 96-px
                                               # images, ragged tail
    (32, 512, 8, 8, 1, 1, 1, 1, 0, 0, 3),      # 1x1, two N tiles
    (64, 256, 9, 9, 1, 1, 1, 1, 0, 0, 2),      # 1x1, odd plane
], ids=lambda c: "x".join(map(str, c)) if isinstance(c, tuple) else c)
def test_tc_both_tile_widths(monkeypatch, case, bn):
    """Every halo kernel (non-persistent N=128; persistent warp-specialised
    N=128 / two stacked 128-pixel sub-tiles / N=256 with TMEM double
    buffering) forced via the plan hooks."""
    monkeypatch.setenv("SMMC_TC_BN", bn[:3])
    monkeypatch.setenv("SMMC_TC_PERSIST", "1" if "p" in bn else "0")
    monkeypatch.setenv("SMMC_TC_MT", "2" if bn.endswith("p2") else "1")
    *gt, n = case
    g = ConvGeometry(*gt)
    x, w, y = _run_tc(g, n, 5)
    samples = [0, n // 2, n - 1]
    ref = orc.smm_conv_c(np.ascontiguousarray(x[samples]), orc.repack(w), g,
                         threads=orc.host_threads())
    err = orc.max_abs_ratio(y[samples], ref)
    assert 1e-5 <= err <= TOL_BF16, err


@pytest.mark.parametrize("split", ["2", "3", "8"])
@pytest.mark.parametrize("case", [(128, 64, 7, 7, 3, 3, 1, 1, 1, 1, 3),
                                  (256, 96, 14, 14, 3, 3, 1, 1, 1, 1, 1),
                                  (64, 40, 9, 11, 1, 1, 1, 1, 0, 0, 2)],
                         ids=lambda c: "x".join(map(str, c)))
def test_tc_split_k(monkeypatch, case, split):
    """Few-tile layers split their channel blocks across CTAs of the
    persistent kernel (fp32 partial planes summed in split order): same
    tolerance, deterministic, and the workspace-less entry runs unsplit."""
    import torch
    from paper_2411_15659_b200 import _native, device
    monkeypatch.setenv("SMMC_TC_SPLIT", split)
    *gt, n = case
    g = ConvGeometry(*gt)
    desc = _native.tc_plan_describe(g, n)
    cblocks = (g.in_channels + 63) // 64
    if cblocks > 1:
        assert "split-K" in desc and device.tc_workspace_bytes(g, n) > 0, desc
    x, w = synthetic_layer(g, n, 17)
    layer = device.TcSmmConv2d(g, w)
    xb = layer.pack_input(torch.from_numpy(x).cuda())
    y1 = layer(xb)
    y2 = layer(xb)
    y0 = device.conv2d_bf16_tc(xb, layer.w_tc, g, workspace=torch.empty(0, dtype=torch.uint8,
                                                                          device="cuda"))
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    for y in (y1, y0):
        assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL_BF16
