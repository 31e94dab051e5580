"""Per-shape autotuning (smmc_autotune_f32): the measured plan choice is one of
the parity-tested plan kinds, so after tuning every layer must still match the
CPU oracle at the fp32 bar, deterministically; clearing restores the default
plan."""

import numpy as np
import pytest

from oracle import smm_oracle as orc
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, _native
from paper_2411_15659_b200.tensors import synthetic_layer

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-4

CASES = [
    # (c_i, c_o, h, w, kh, kw, sh, sw, ph, pw), n
    ((192, 384, 13, 13, 3, 3, 1, 1, 1, 1), 1),     # AlexNet conv3 at the harness batch of 1
    ((3, 64, 67, 67, 11, 11, 4, 4, 0, 0), 1),      # 11x11 s4 stem, one small sample
    ((256, 128, 13, 13, 1, 1, 1, 1, 0, 0), 1),     # YOLOv3-tiny 1x1
    ((64, 192, 27, 27, 5, 5, 1, 1, 2, 2), 2),      # AlexNet conv2 (5x5 tap-major)
    ((24, 37, 11, 9, 3, 3, 1, 1, 1, 1), 3),        # ragged, generic K order
]


@pytest.fixture(autouse=True)
def _clear():
    _native.autotune_clear()
    yield
    _native.autotune_clear()


@pytest.mark.parametrize("gt,n", CASES, ids=lambda v: str(v))
def test_autotuned_plan_matches_oracle(gt, n):
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(*gt)
    default_desc = _native.plan_describe(g, n)
    x, w = synthetic_layer(g, n, 19)
    xd = torch.from_numpy(x).cuda()
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    y_default = device.conv2d(xd, wd, g)
    report = _native.autotune(g, n, iters=5)
    assert report.startswith("default "), report
    tuned_desc = _native.plan_describe(g, n)
    assert ("kept plan" in report) == (tuned_desc != default_desc), (report, default_desc, tuned_desc)
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, report
    assert orc.max_abs_ratio(y_default.cpu().numpy(), ref) <= TOL_FP32
    # the host-buffer entry sizes its workspace from the tuned plan
    yh = smm.smm_conv_batched(x, smm.repack_weights(w, g), g)
    assert orc.max_abs_ratio(yh, ref) <= TOL_FP32
    _native.autotune_clear()
    assert _native.plan_describe(g, n) == default_desc


def test_autotune_keeps_other_shapes_and_batches_untouched():
    g = ConvGeometry(192, 384, 13, 13, 3, 3, 1, 1, 1, 1)
    other = ConvGeometry(128, 128, 28, 28, 3, 3, 1, 1, 1, 1)
    d_other, d_n4 = _native.plan_describe(other, 1), _native.plan_describe(g, 4)
    _native.autotune(g, 1, iters=3)
    assert _native.plan_describe(other, 1) == d_other
    assert _native.plan_describe(g, 4) == d_n4


def test_fitted_layer_autotunes_on_request():
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(384, 256, 13, 13, 3, 3, 1, 1, 1, 1)
    x, w = synthetic_layer(g, 1, 3)
    mod = device.SmmConv2d(g, w, max_batch=1, autotune=True)
    assert mod.autotune_report and mod.autotune_report.startswith("default ")
    y = mod(torch.from_numpy(x).cuda())
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL_FP32
