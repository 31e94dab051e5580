"""GPU parity of the direct stem kernel (csrc/conv_stem.cu): c_i <= 4 layers
with 3x3 s1, 7x7 s2 and 11x11 s4 kernels — VGG conv1_1 and the BASELINE
config-3 stems plus ragged geometries (odd widths, partial 8-column
groups, c_o not a multiple of 4, unequal strides and pads, 1-row planes) —
against the CPU oracle at the fp32 bar, deterministic, and against the tiled
kernel it replaces (SMMC_STEM=0)."""

import numpy as np
import pytest

from oracle import smm_oracle as orc
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, _native
from paper_2411_15659_b200.tensors import synthetic_layer

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-4

STEM_CASES = [
    # (c_i, c_o, h, w, kh, kw, sh, sw, ph, pw), n
    ((3, 64, 224, 224, 3, 3, 1, 1, 1, 1), 1),      # VGG conv1_1 (config 4), one sample
    ((3, 64, 224, 224, 7, 7, 2, 2, 3, 3), 1),      # config 3 7x7 s2 stem
    ((1, 5, 13, 17, 3, 3, 2, 1, 1, 1), 2),         # 3x3, s_h != s_w, c_o % 4 != 0
    ((3, 16, 9, 9, 3, 3, 1, 1, 1, 1), 3),          # w' = 9: one full + one 1-column group
    ((4, 130, 12, 30, 3, 3, 1, 1, 0, 1), 2),       # 3x3, three channel tiles, unequal pads
    ((3, 96, 227, 227, 11, 11, 4, 4, 0, 0), 2),    # config 3 11x11 s4 stem (w' = 55)
    ((3, 40, 47, 47, 11, 11, 4, 4, 0, 0), 3),      # c_o < tile, ragged
    ((1, 5, 13, 17, 7, 7, 2, 2, 3, 3), 2),         # c_o % 4 != 0, one channel
    ((4, 70, 30, 30, 7, 7, 1, 2, 2, 3), 2),        # s_h != s_w, unequal pads, two channel tiles
    ((2, 3, 9, 10, 7, 7, 3, 2, 3, 3), 3),          # s_h = 3, tiny plane
    ((3, 16, 9, 39, 7, 7, 2, 2, 3, 3), 3),         # w' = 20: partial 8-column group
    ((3, 8, 1, 40, 7, 7, 1, 2, 3, 0), 2),          # 1-row input, unequal pads
    ((3, 33, 40, 40, 11, 11, 4, 4, 0, 0), 1),      # no padding, c_o % 4 != 0
    ((2, 12, 20, 31, 11, 11, 4, 4, 5, 2), 2),      # pads on the strided stem
]


def _run(g, n, seed):
    import torch
    from paper_2411_15659_b200 import device
    x, w = synthetic_layer(g, n, seed)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    return x, w, xd, wd, device


@pytest.mark.parametrize("gt,n", STEM_CASES, ids=lambda v: str(v))
def test_stem_kernel_matches_oracle(gt, n, monkeypatch):
    import torch
    g = ConvGeometry(*gt)
    monkeypatch.setenv("SMMC_STEM", "1")   # the stem kernel at any size (small problems plan tiled)
    desc = _native.plan_describe(g, n)
    assert "direct stem" in desc, desc
    x, w, xd, wd, device = _run(g, n, 7)
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    monkeypatch.setenv("SMMC_STEM", "0")
    assert "direct stem" not in _native.plan_describe(g, n)
    yt = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2), desc
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, desc
    assert orc.max_abs_ratio(yt.cpu().numpy(), ref) <= TOL_FP32


def test_stem_kernel_on_unaligned_input_and_host_entry(monkeypatch):
    """x at an odd 4-byte offset (a sample slice of an odd-sized batch) and
    the host-buffer entry point (chunked pipeline) both reach the stem kernel."""
    import ctypes
    import torch
    monkeypatch.setenv("SMMC_STEM", "1")
    g = ConvGeometry(3, 64, 31, 31, 7, 7, 2, 2, 3, 3)
    x, w = synthetic_layer(g, 3, 11)
    ws = smm.repack_weights(w, g)
    wsd = torch.from_numpy(ws).cuda()
    xd = torch.from_numpy(x).cuda().reshape(-1)
    lib = _native.lib()
    G = _native.Geom.of(g, 2)
    y = torch.empty((2,) + g.output_shape, device="cuda")
    per = g.in_channels * g.in_h * g.in_w  # odd number of floats
    _native.check(lib.smmc_conv2d_fwd_f32(ctypes.c_void_p(xd.data_ptr() + 4 * per),
                                          ctypes.c_void_p(wsd.data_ptr()),
                                          ctypes.c_void_p(y.data_ptr()),
                                          ctypes.byref(G), 0, None, 0, None), "conv")
    torch.cuda.synchronize()
    ref = orc.smm_conv_c(np.ascontiguousarray(x[1:]), ws, g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL_FP32
    yh = smm.smm_conv_batched(np.ascontiguousarray(x[1:]), ws, g)
    assert orc.max_abs_ratio(yh, ref) <= TOL_FP32


def test_random_stem_geometries(monkeypatch):
    """80 random c_i <= 4 geometries over the stem kernel's tap kinds; other
    c_i <= 4 kernels (5x5, ...) stay on the tiled kernel."""
    import torch
    monkeypatch.setenv("SMMC_STEM", "1")
    rng = np.random.default_rng(31337)
    kinds = [(3, 3, 1), (7, 7, 2), (11, 11, 4)]
    checked = 0
    while checked < 80:
        kh, kw, sw = kinds[int(rng.integers(0, 3))]
        ci = int(rng.integers(1, 5))
        co = int(rng.integers(1, 140))
        h, wd_ = int(rng.integers(1, 60)), int(rng.integers(1, 60))
        sh = int(rng.integers(1, 5))
        ph, pw = int(rng.integers(0, kh // 2 + 1)), int(rng.integers(0, kw // 2 + 1))
        if kh > h + 2 * ph or kw > wd_ + 2 * pw:
            continue
        g = ConvGeometry(ci, co, h, wd_, kh, kw, sh, sw, ph, pw)
        n = int(rng.integers(1, 4))
        checked += 1
        assert "direct stem" in _native.plan_describe(g, n), g
        x, w, xd, wdev, device = _run(g, n, checked)
        y = device.conv2d(xd, wdev, g)
        torch.cuda.synchronize()
        ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
        assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL_FP32, (g, n)


def test_other_small_channel_layers_stay_on_the_tiled_kernel():
    for gt in [(3, 16, 20, 20, 5, 5, 1, 1, 2, 2), (5, 64, 40, 40, 7, 7, 2, 2, 3, 3),
               (8, 64, 40, 40, 3, 3, 1, 1, 1, 1), (3, 16, 20, 20, 3, 3, 1, 2, 1, 1)]:
        assert "direct stem" not in _native.plan_describe(ConvGeometry(*gt), 2), gt


# c_i = 3, 3x3 s1 p_w = 1 layers with 16-byte rows run the resident-window
# kernel (conv_stem_rw_kernel: channel passes over one window set, cross-tile
# prefetch, strided tile walk): tile tails in every dimension of that walk.
RW_CASES = [
    # (c_i, c_o, h, w, kh, kw, sh, sw, ph, pw), n
    ((3, 64, 224, 224, 3, 3, 1, 1, 1, 1), 2),   # VGG conv1_1, two samples (n carry)
    ((3, 64, 12, 16, 3, 3, 1, 1, 1, 1), 5),     # fewer tiles than threads in the grid
    ((3, 16, 20, 8, 3, 3, 1, 1, 1, 1), 3),      # c_o < one pass: scalar epilogue
    ((3, 40, 9, 12, 3, 3, 1, 1, 1, 1), 2),      # c_o tail inside the second pass
    ((3, 132, 10, 20, 3, 3, 1, 1, 0, 1), 2),    # three channel tiles, no row padding
    ((3, 64, 7, 4, 3, 3, 2, 1, 1, 1), 4),       # one column group per row, s_h = 2
    ((3, 128, 64, 256, 3, 3, 1, 1, 1, 1), 1),   # wide rows, two channel tiles
    ((3, 64, 1, 36, 3, 3, 1, 1, 1, 1), 7),      # 1-row planes: every window row is padding but one
    ((3, 96, 8, 16, 3, 3, 1, 1, 1, 1), 2),      # c_o = 96: three 32-channel CTAs, one pass each
    ((3, 16, 416, 416, 3, 3, 1, 1, 1, 1), 1),   # YOLOv3-tiny conv1: one 16-channel group per warp
]


@pytest.mark.parametrize("gt,n", RW_CASES, ids=lambda v: str(v))
def test_resident_window_stem_matches_oracle_and_round1_kernel(gt, n, monkeypatch):
    import torch
    g = ConvGeometry(*gt)
    assert "direct stem" in _native.plan_describe(g, n)
    x, w, xd, wd, device = _run(g, n, 23)
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    monkeypatch.setenv("SMMC_STEM_RW0", "1")   # the round-1 stem kernel: same (c, kh, kw) order
    y0 = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert torch.equal(y1, y0), "resident-window kernel differs from the round-1 stem kernel"
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32


def test_resident_window_stem_large_batch_linearity():
    """Whole conv1_1 batch of config 4 at a reduced N: conv(2x) == 2 conv(x)
    exactly and every sample equals sample-by-sample launches (the strided
    walk crosses samples)."""
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(3, 64, 224, 224, 3, 3, 1, 1, 1, 1)
    x, w = synthetic_layer(g, 16, 5)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    y = device.conv2d(xd, wd, g)
    y2 = device.conv2d(2 * xd, wd, g)
    assert torch.equal(y2, 2 * y)
    for i in (0, 7, 15):
        yi = device.conv2d(xd[i:i + 1].contiguous(), wd, g)
        assert torch.equal(yi[0], y[i])
