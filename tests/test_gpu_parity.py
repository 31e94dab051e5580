"""GPU parity: the sm_100a kernels, called through the C ABI, against the
reference's own outputs (golden vectors) and the CPU oracle.

Bars (BASELINE.json): exact mode bitwise; FFMA mode
max|y - ref| <= 1e-4 * max|ref| (float64 metric).
"""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, GOLDEN_SLICES
from oracle import smm_oracle as orc
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, ShapeMismatchError, _native
from paper_2411_15659_b200.tensors import synthetic_layer
from paper_2411_15659_b200.workloads import CONFIGS, layer_seed

pytestmark = pytest.mark.gpu

TOL_FP32 = 1e-4


@pytest.mark.parametrize("case", GOLDEN_CASES, ids=lambda c: c.name)
def test_exact_mode_bitwise_vs_reference(case):
    ws = smm.repack_weights(case.w, case.geom)
    y = smm.smm_conv_batched(np.ascontiguousarray(case.x), ws, case.geom, mode="exact")
    assert np.array_equal(y, case.y_smm), case.name


@pytest.mark.parametrize("case", GOLDEN_CASES, ids=lambda c: c.name)
def test_ffma_mode_within_tolerance(case):
    ws = smm.repack_weights(case.w, case.geom)
    y = smm.smm_conv_batched(np.ascontiguousarray(case.x), ws, case.geom, mode="ffma")
    assert orc.max_abs_ratio(y, case.y_smm) <= TOL_FP32, case.name
    if case.kind == "kat":
        assert np.array_equal(y, case.y_smm)


def test_single_and_parallel_entry_points():
    case = next(c for c in GOLDEN_CASES if c.name == "cfg2_3x3_c24_14")
    ws = smm.repack_weights(case.w, case.geom)
    x0 = np.ascontiguousarray(case.x[0])
    single = smm.smm_conv_single(x0, ws, case.geom)
    assert single.shape == case.geom.output_shape
    assert orc.max_abs_ratio(single, case.y_smm[0]) <= TOL_FP32
    assert np.array_equal(smm.smm_conv_single(x0, ws, case.geom, fused=False), single)
    for d in (1, 2, 3, 4, 7, 8, 16):
        assert np.array_equal(smm.smm_conv_parallel(x0, ws, case.geom, d), single)
    exact = smm.smm_conv_single(x0, ws, case.geom, mode="exact")
    assert np.array_equal(exact, case.y_smm[0])
    with pytest.raises(ValueError):
        smm.smm_conv_parallel(x0, ws, case.geom, 0)


def test_boundary_errors_before_compute():
    g = ConvGeometry(2, 3, 6, 6, 3, 3)
    x = np.zeros(g.input_shape, np.float32)
    w = np.zeros(g.weights_shape, np.float32)
    with pytest.raises(ShapeMismatchError):
        smm.smm_conv_single(x, w, g)  # not repacked
    with pytest.raises(ShapeMismatchError):
        smm.smm_conv_single(x.astype(np.float64), smm.repack_weights(w, g), g)
    with pytest.raises(ShapeMismatchError):
        smm.smm_conv_single(np.asfortranarray(np.zeros((2, 6, 6), np.float32)),
                            smm.repack_weights(w, g), g)


def test_extract_slice_and_fma_helpers(golden_data):
    g = ConvGeometry(*GOLDEN_SLICES["geom"])
    x = golden_data["slices__x"]
    for c in range(g.in_channels):
        for j in range(g.k_w):
            buf = np.empty((g.padded_h, g.out_w), np.float32)
            smm.extract_slice(x, g, c, j, buf)
            assert np.array_equal(buf, golden_data[f"slices__c{c}_j{j}"])
            for k in range(g.k_h):
                view = smm.shifted_view(buf, k, g)
                assert np.shares_memory(view, buf)
    src = smm.random_tensor((5, 7), 3)
    dst = smm.random_tensor((5, 7), 4)
    expect = dst + np.float32(0.377) * src
    smm.scalar_matrix_fma(0.377, src, dst)
    assert np.array_equal(dst, expect)
    # strided source view (test_smm.py:153-160)
    g2 = ConvGeometry(1, 1, 8, 4, 3, 3, stride_h=2)
    buf = np.arange(g2.padded_h * g2.out_w, dtype=np.float32).reshape(g2.padded_h, g2.out_w)
    view = smm.shifted_view(buf, 1, g2)
    out = np.zeros((g2.out_h, g2.out_w), np.float32)
    smm.scalar_matrix_fma(2.0, view, out)
    assert np.array_equal(out, 2.0 * view)


def _device_run(g, n, seed, mode="ffma"):
    import torch
    from paper_2411_15659_b200 import device
    x, w = synthetic_layer(g, n, seed)
    xd = torch.from_numpy(x).cuda()
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    y = device.conv2d(xd, wd, g, mode=mode)
    torch.cuda.synchronize()
    return x, w, y


def _check_samples(x, w, g, y, samples):
    ws = orc.repack(w)
    ref = orc.smm_conv_c(np.ascontiguousarray(x[samples]), ws, g, threads=orc.host_threads())
    err = orc.max_abs_ratio(y[samples], ref)
    assert err <= TOL_FP32, err
    return err


LAYERS = [(ci, li, name, n, g) for ci, cfg in CONFIGS.items()
          for li, (name, n, g) in enumerate(cfg["layers"])]


@pytest.mark.parametrize("ci,li,name,n,g", LAYERS, ids=[l[2] + f"_cfg{l[0]}" for l in LAYERS])
def test_baseline_layer_parity_full_size(ci, li, name, n, g):
    """Every BASELINE.json layer at full size.  All samples are checked
    against the oracle when cheap; for big batches the first and last sample
    (samples are independent, estimator.py:123-124) plus a size-independent
    linearity property over the whole batch."""
    import torch
    x, w, y = _device_run(g, n, layer_seed(ci, li))
    yh = y.cpu().numpy()
    assert np.isfinite(yh).all()
    per_sample_gflop = g.flops(1) / 1e9
    samples = list(range(n)) if n * per_sample_gflop <= 2.0 else [0, n - 1]
    _check_samples(x, w, g, yh, samples)
    # linearity over the whole batch: conv(a*x) == a*conv(x) for a power of two
    # is exact in fp32 (scaling by 2 commutes with every rounding).
    from paper_2411_15659_b200 import device
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    y2 = device.conv2d(torch.from_numpy(x).cuda() * 2.0, wd, g)
    assert torch.equal(y2, y * 2.0)
    # determinism: identical bits on a second launch
    y3 = device.conv2d(torch.from_numpy(x).cuda(), wd, g)
    assert torch.equal(y3, y)


def test_exact_mode_bitwise_at_config1_full_size():
    g = CONFIGS[1]["layers"][0][2]
    x, w, y = _device_run(g, 1, layer_seed(1, 0), mode="exact")
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert np.array_equal(y.cpu().numpy(), ref)


def test_batch_composition_and_empty_batch():
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(32, 48, 14, 14, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 9, 77)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    full = device.conv2d(xd, wd, g)
    parts = torch.cat([device.conv2d(xd[i:i + 3].contiguous(), wd, g) for i in (0, 3, 6)])
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(full.cpu().numpy(), ref) <= TOL_FP32
    assert orc.max_abs_ratio(parts.cpu().numpy(), ref) <= TOL_FP32
    empty = device.conv2d(xd[:0], wd, g)
    assert empty.shape == (0,) + g.output_shape


def test_device_path_rejects_bad_tensors():
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(4, 8, 10, 10, 3, 3)
    w = torch.zeros(g.weights_smm_shape, device="cuda")
    with pytest.raises(ShapeMismatchError):
        device.conv2d(torch.zeros((1,) + g.input_shape), w, g)  # CPU tensor
    with pytest.raises(ShapeMismatchError):
        device.conv2d(torch.zeros((1,) + g.input_shape, device="cuda", dtype=torch.float64), w, g)
    with pytest.raises(ShapeMismatchError):
        device.conv2d(torch.zeros((1, 4, 10, 11), device="cuda"), w, g)


def test_split_k_and_fused_plans_both_exercised():
    g_small = ConvGeometry(512, 512, 7, 7, 3, 3, pad_h=1, pad_w=1)
    g_big = ConvGeometry(64, 128, 112, 112, 3, 3, pad_h=1, pad_w=1)
    # N=1 512@7: split-K reduced inside the one launch (reduce mode 5)
    assert _native.plan_launches(g_small, 1) == 1
    assert "in-kernel" in _native.plan_describe(g_small, 1)
    assert _native.workspace_bytes(g_small, 1) > 0
    assert _native.plan_launches(g_big, 64) == 1
    assert _native.workspace_bytes(g_big, 64) == 0


def test_estimator_transform():
    from paper_2411_15659_b200 import Conv2D
    X = smm.random_tensor((3, 2, 8, 8), 0)
    est = Conv2D(out_channels=4, kernel_size=3, padding=1).fit(X)
    out = est.transform(X)
    assert out.shape == (3, 4, 8, 8) and out.dtype == np.float32
    ref = orc.smm_conv_c(X, est.weights_smm_, est.geometry_)
    assert orc.max_rel_diff(out, ref) <= 1e-4
    a = Conv2D(out_channels=3, kernel_size=3, threads=1).fit(X).transform(X)
    b = Conv2D(out_channels=3, kernel_size=3, threads=3).fit(X).transform(X)
    assert np.array_equal(a, b)
    exact = Conv2D(out_channels=4, kernel_size=3, padding=1, backend="smm_exact").fit(X)
    assert np.array_equal(exact.transform(X), ref)
    weights = np.zeros((1, 1, 3, 3), np.float32)
    weights[0, 0, 1, 1] = 2.0
    X1 = smm.random_tensor((1, 1, 6, 6), 6)
    out = Conv2D(out_channels=1, kernel_size=3, weights=weights).fit(X1).transform(X1)
    assert np.array_equal(out[0, 0], 2.0 * X1[0, 0, 1:5, 1:5])


def test_launch_counter_and_plan_describe():
    g = ConvGeometry(64, 64, 56, 56, 3, 3, pad_h=1, pad_w=1)
    before = _native.launch_count()
    import torch
    from paper_2411_15659_b200 import device
    x = torch.zeros((2,) + g.input_shape, device="cuda")
    w = torch.zeros(g.weights_smm_shape, device="cuda")
    device.conv2d(x, w, g)
    torch.cuda.synchronize()
    assert _native.launch_count() - before == _native.plan_launches(g, 2)
    assert "ffma" in _native.plan_describe(g, 2)


@pytest.mark.parametrize("cluster", ["1", "0"])
@pytest.mark.parametrize("plan", ["0,1", "0,3", "1,2", "1,0", "2,0", "3,0", "3,8", "1,24", "0,0",
                                  "2,5", "3,7"])
def test_every_reduction_mode_matches_oracle(plan, cluster, monkeypatch):
    """Force each work decomposition (no split, split-K reduced in a cluster
    through DSMEM / by the last arriver / by a reduce kernel, stream-K) on one
    geometry: all within tolerance of the oracle, each bitwise deterministic
    across launches."""
    import torch
    from paper_2411_15659_b200 import device
    monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
    monkeypatch.setenv("SMMC_CLUSTER_RED", cluster)
    g = ConvGeometry(64, 96, 20, 20, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 6, 123)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    desc = _native.plan_describe(g, 6)
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2), desc
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, desc
    if plan.endswith(",0"):
        assert "stream-K" in desc
    if cluster == "0":
        assert "cluster" not in desc, desc


@pytest.mark.parametrize("cluster", ["1", "0"])
@pytest.mark.parametrize("plan", ["5,1", "5,2", "5,3", "5,8", "5,36", "5,4,1,5", "5,7,1,5"])
@pytest.mark.parametrize("gt,n", [((64, 32, 20, 20, 3, 3, 1, 1, 1, 1), 5),     # c_o = 32: one channel tile
                                  ((32, 88, 17, 23, 5, 5, 1, 1, 2, 2), 2),     # c_o % 64 = 24, ragged pixels
                                  ((16, 7, 30, 30, 3, 3, 2, 2, 0, 1), 3)])     # c_o % 4 != 0, strided
def test_narrow_channel_tile_every_reduction(gt, n, plan, cluster, monkeypatch):
    """The 128 x 32 tile (64 threads, two pixel columns per loader thread) under
    no split, last arriver / cluster DSMEM, reduce kernel and in-kernel split
    reductions: oracle parity, bitwise run to run."""
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(*gt)
    monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
    monkeypatch.setenv("SMMC_CLUSTER_RED", cluster)
    desc = _native.plan_describe(g, n)
    assert "tile 128x32" in desc, desc
    x, w = synthetic_layer(g, n, 77)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2), desc
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, desc


@pytest.mark.parametrize("cluster", ["1", "0"])
@pytest.mark.parametrize("plan", ["1,1,4", "3,1,2", "0,1,2", "1,3,2", "1,8,4", "3,6,4", "1,16,4",
                                  "3,32,2", "0,12,2", "1,4,3", "3,5,3"])
def test_warp_group_split_matches_oracle(plan, cluster, monkeypatch):
    """Warp-group split-K (G groups per CTA over the CTA's tap blocks, partial
    tiles summed in group order through shared memory) under every outer
    reduction (none, last arriver, cluster DSMEM, reduce kernel), including
    groups left without tap blocks: oracle parity, bitwise run to run."""
    import torch
    from paper_2411_15659_b200 import device
    monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
    monkeypatch.setenv("SMMC_CLUSTER_RED", cluster)
    g = ConvGeometry(64, 96, 20, 20, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 3, 321)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    desc = _native.plan_describe(g, 3)
    assert "warp groups" in desc, desc
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2), desc
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, desc


@pytest.mark.parametrize("plan", ["1,2", "1,8", "3,5", "0,3"])
def test_cluster_dsmem_split_reduction(plan, monkeypatch):
    """Under-filled split-K grids reduce their partial tiles inside a
    thread-block cluster through distributed shared memory (one kernel, no
    workspace); ragged tiles and c_o % 4 != 0 included."""
    monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
    for g, n in ((ConvGeometry(48, 70, 11, 9, 3, 3, pad_h=1, pad_w=1), 1),
                 (ConvGeometry(32, 64, 12, 12, 3, 3, pad_h=1, pad_w=1), 2)):
        desc = _native.plan_describe(g, n)
        assert "cluster" in desc and _native.workspace_bytes(g, n) == 0, desc
        assert _native.plan_launches(g, n) == 1
        x, w = synthetic_layer(g, n, 77)
        ws = smm.repack_weights(w, g)
        y = smm.smm_conv_batched(x, ws, g)
        assert np.array_equal(y, smm.smm_conv_batched(x, ws, g))
        ref = orc.smm_conv_c(x, orc.repack(w), g)
        assert orc.max_abs_ratio(y, ref) <= TOL_FP32, desc


def _draw(rng):
    """A random small geometry over the reference acceptance sweep's ranges
    (test_acceptance.py:51-68): c in [1, 8], h, w in [4, 32], k in {1,3,5,7},
    stride in {1, 2}, pad in {0, 1, 2}; None when the kernel does not fit."""
    ci, co = int(rng.integers(1, 9)), int(rng.integers(1, 9))
    h, w = int(rng.integers(4, 33)), int(rng.integers(4, 33))
    kh, kw = int(rng.choice((1, 3, 5, 7))), int(rng.choice((1, 3, 5, 7)))
    sh, sw = int(rng.choice((1, 2))), int(rng.choice((1, 2)))
    ph, pw = int(rng.choice((0, 1, 2))), int(rng.choice((0, 1, 2)))
    if kh > h + 2 * ph or kw > w + 2 * pw:
        return None
    return ConvGeometry(ci, co, h, w, kh, kw, sh, sw, ph, pw)


def test_acceptance_sweep_200_random_geometries():
    """The reference's acceptance criterion 1 on the GPU: 200 random
    geometries (seed 20240601), splitmix64 data, FFMA mode within
    max_rel_diff 1e-4 of the oracle, exact mode bitwise, batches of 1-3
    samples, and bitwise launch-to-launch determinism."""
    from paper_2411_15659_b200.tensors import random_tensor
    rng = np.random.default_rng(20240601)
    checked, worst = 0, 0.0
    while checked < 200:
        g = _draw(rng)
        if g is None:
            continue
        checked += 1
        n = 1 + checked % 3
        x = random_tensor((n,) + g.input_shape, 2 * checked)
        w = random_tensor(g.weights_shape, 2 * checked + 1)
        ws = smm.repack_weights(w, g)
        ref = orc.smm_conv_c(x, orc.repack(w), g)
        y = smm.smm_conv_batched(x, ws, g)
        d = orc.max_rel_diff(y, ref)
        worst = max(worst, d)
        assert d <= 1e-4, (g, d)
        assert np.array_equal(smm.smm_conv_batched(x, ws, g), y), g
        assert np.array_equal(smm.smm_conv_batched(x, ws, g, mode="exact"), ref), g
    assert worst > 0.0  # the FFMA path really reorders the sums


@pytest.mark.parametrize("gt,n,narrow", [((64, 256, 56, 56, 1, 1), 3, 0), ((256, 64, 28, 28, 1, 1), 2, 0),
                                         ((48, 100, 6, 10, 1, 1), 3, 0), ((16, 4, 4, 4, 1, 1), 1, 0),
                                         ((64, 48, 6, 6, 1, 1), 3, 2), ((64, 64, 56, 56, 1, 1), 16, 2),
                                         ((256, 64, 28, 28, 1, 1), 2, 2), ((64, 48, 18, 18, 1, 1), 15, 1),
                                         ((256, 64, 56, 56, 1, 1), 8, 1), ((384, 64, 14, 14, 1, 1), 25, 1)],
                         ids=["64to256", "256to64", "ragged", "tiny", "warp_tile_forced_ragged",
                              "warp_tile_forced_multi_tile_warps", "warp_tile_forced_one_warp",
                              "warp_tile_ragged_3_per_sm", "config3_256to64", "warp_tile_384_2_per_sm"])
@pytest.mark.parametrize("wres", ["1", "0"], ids=["weights_resident", "weights_streamed"])
def test_persistent_1x1_matches_tiled_kernel_bitwise(gt, n, narrow, wres, monkeypatch):
    """1x1 layers run a persistent block-stream kernel (the weight slice
    resident in shared memory, or streamed with the input; for c_o <= 64 on
    grids of 2-12 warp tiles per SM, warp tiles with private rings): same summation
    order as the tiled kernel (bitwise equal to it), oracle parity, and the
    tiled fallback for operands that are not 16-byte aligned."""
    import torch
    from paper_2411_15659_b200 import device
    monkeypatch.setenv("SMMC_1X1_WRES", wres)
    if narrow == 2:  # the c_o <= 64 warp-tile kernel outside the shapes its rule picks
        if wres == "0":
            pytest.skip("one run of the forced warp-tile cases is enough")
        monkeypatch.setenv("SMMC_1X1_NARROW", "2")
    g = ConvGeometry(*gt)
    desc = _native.plan_describe(g, n)
    assert "persistent 1x1" in desc
    assert ("warp-tile" in desc) == (narrow > 0)
    x, w = synthetic_layer(g, n, 99)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    y = device.conv2d(xd, wd, g)
    buf = torch.empty(x.size + 1, device="cuda")
    xm = buf[1:].view(x.shape)
    xm.copy_(xd)
    ym = device.conv2d(xm, wd, g)  # 4-byte aligned input: tiled fallback
    # the tiled kernel on the same tile without split-K (same summation order)
    monkeypatch.setenv("SMMC_FORCE_PLAN", "1,1" if g.out_channels <= 64 else "3,1")
    assert "persistent" not in _native.plan_describe(g, n)
    yt = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y, yt) and torch.equal(y, ym)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL_FP32


@pytest.mark.parametrize("plan", ["1,0", "2,0", "0,0", "3,0"])
@pytest.mark.parametrize("gt,n", [((3, 64, 40, 40, 7, 7, 2, 2, 3, 3), 3),
                                  ((3, 40, 47, 47, 11, 11, 4, 4, 0, 0), 2),
                                  ((5, 24, 19, 23, 3, 5, 1, 2, 1, 2), 2)],
                         ids=["7x7s2", "11x11s4", "ragged"])
def test_stream_k_on_the_generic_k_order(gt, n, plan, monkeypatch):
    """Stream-K over the reference's (c, j, k) update order (the c_i = 3 stems
    and any c_i % 16 != 0 layer): oracle parity, deterministic."""
    import torch
    from paper_2411_15659_b200 import device
    monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
    g = ConvGeometry(*gt)
    desc = _native.plan_describe(g, n)
    assert "stream-K" in desc and "(c,j,k)" in desc, desc
    x, w = synthetic_layer(g, n, 5)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda()
    y1 = device.conv2d(xd, wd, g)
    y2 = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2), desc
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, desc


def test_random_geometries_wide_channels():
    """150 random geometries beyond the reference's small-channel acceptance
    ranges: c_i multiples of 16 (the tap-major K order, 16-byte weight rows)
    and ragged c_o, planes 1-40 wide, kernels 1-5, strides 1-2, batches 1-6 —
    whatever plan the planner picks (split-K, cluster DSMEM, reduce kernel,
    stream-K, warp groups, the persistent 1x1 kernel), within the fp32 bar of
    the oracle (BASELINE signed data) and bitwise deterministic."""
    import torch
    from paper_2411_15659_b200 import device
    rng = np.random.default_rng(424242)
    checked = 0
    plans = set()
    while checked < 150:
        ci = int(rng.choice((16, 32, 48, 64, 96, 128)))
        co = int(rng.integers(1, 200))
        h, w = int(rng.integers(1, 41)), int(rng.integers(1, 41))
        k = int(rng.choice((1, 3, 5)))
        s = int(rng.choice((1, 1, 2)))
        p = int(rng.choice((0, 1, 2)))
        if k > h + 2 * p or k > w + 2 * p:
            continue
        g = ConvGeometry(ci, co, h, w, k, k, s, s, p, p)
        n = int(rng.integers(1, 7))
        checked += 1
        x, wt = synthetic_layer(g, n, checked)
        wd = torch.from_numpy(smm.repack_weights(wt, g)).cuda()
        xd = torch.from_numpy(x).cuda()
        y1 = device.conv2d(xd, wd, g)
        y2 = device.conv2d(xd, wd, g)
        torch.cuda.synchronize()
        desc = _native.plan_describe(g, n)
        plans.add(desc.split("reduce=")[-1].split(")")[0])
        assert torch.equal(y1, y2), (g, n, desc)
        ref = orc.smm_conv_c(x, orc.repack(wt), g, threads=orc.host_threads())
        assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, (g, n, desc)
    assert len(plans) >= 3, plans  # several reduction schemes were exercised


@pytest.mark.parametrize("plan", ["4,3,4,5", "4,9,4,5", "4,18,2,5", "1,4,1,5", "3,5,2,5", "0,6,1,5",
                                  "4,32,1,5", "1,16,2,5"])
def test_in_kernel_split_reduction(plan, monkeypatch):
    """Reduce mode 5: all S split CTAs of a tile (cooperative grid) publish
    their partial tiles, wait on the tile counter and each sums a slice in
    split order -- S beyond the cluster limit, warp groups, ragged tiles and
    7x7 planes (h'*w' % 4 != 0).  Oracle parity, bitwise run to run, and the
    counters re-armed: the same zero-at-rest workspace serves other layers
    and plans in between."""
    import torch
    from paper_2411_15659_b200 import device
    monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
    ws = None
    for g, n in ((ConvGeometry(64, 96, 20, 20, 3, 3, pad_h=1, pad_w=1), 1),
                 (ConvGeometry(128, 72, 7, 7, 3, 3, pad_h=1, pad_w=1), 2),
                 (ConvGeometry(64, 64, 9, 11, 3, 3, pad_h=1, pad_w=1), 1)):
        desc = _native.plan_describe(g, n)
        assert "in-kernel" in desc and _native.plan_launches(g, n) == 1, desc
        x, w = synthetic_layer(g, n, 91)
        wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
        xd = torch.from_numpy(x).cuda()
        need = _native.workspace_bytes(g, n)
        if ws is None or ws.numel() < need:
            ws = torch.zeros(max(need, 1 << 22), dtype=torch.uint8, device="cuda")
        y1 = device.conv2d(xd, wd, g, workspace=ws)
        y2 = device.conv2d(xd, wd, g, workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(y1, y2), desc
        ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
        assert orc.max_abs_ratio(y1.cpu().numpy(), ref) <= TOL_FP32, desc
    # the counter region is zero again after the launches
    assert int(ws[: 64 * 1024].count_nonzero()) == 0


def test_workspace_counter_region_shared_across_plans(monkeypatch):
    """One zero-initialised workspace reused by a last-arriver plan, a
    stream-K plan, a reduce-kernel plan and an in-kernel plan in turn (no
    per-call zeroing): every result matches the oracle."""
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(64, 96, 14, 14, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 2, 17)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(smm.repack_weights(w, g)).cuda()
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(2):
        for plan in ("1,3", "3,0", "1,8", "4,6,2,5", "1,2", "0,4,1,5"):
            monkeypatch.setenv("SMMC_FORCE_PLAN", plan)
            monkeypatch.setenv("SMMC_CLUSTER_RED", "0")
            y = device.conv2d(xd, wd, g, workspace=ws)
            torch.cuda.synchronize()
            assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL_FP32, (plan, rep)
    assert int(ws[: 64 * 1024].count_nonzero()) == 0
