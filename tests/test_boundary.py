"""The C-ABI library: it loads, exports every symbol include/smmc.h declares,
and its host-side logic (geometry checks, plans, error mapping) works without
a GPU — while compute without a GPU fails loudly (no CPU fallback)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, DeviceError, GeometryError, _native

HEADER = Path(__file__).resolve().parents[1] / "include" / "smmc.h"


def _declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^SMMC_API\s+[\w\s\*]+?\b(smmc_\w+)\(", text, re.M)))


def test_header_and_binding_agree():
    assert _declared() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    lib = _native.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert lib.smmc_abi_version() == 1


def test_symbols_visible_in_dynamic_table():
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (smmc_\w+)", out))
    assert set(_declared()) <= exported
    # nothing but the ABI is exported with default visibility from our code
    assert all(s.startswith("smmc_") for s in exported)


def test_sm100a_cubin_embedded():
    import subprocess
    cuobjdump = "/usr/local/cuda/bin/cuobjdump"
    if not Path(cuobjdump).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_geom_check_mirrors_python_geometry():
    lib = _native.lib()
    oh, ow = ctypes.c_int32(), ctypes.c_int32()
    g = _native.Geom(1, 3, 227, 227, 96, 11, 11, 4, 4, 0, 0)
    assert lib.smmc_geom_check(ctypes.byref(g), ctypes.byref(oh), ctypes.byref(ow)) == 0
    assert (oh.value, ow.value) == (55, 55)
    for bad in [(1, 0, 4, 4, 1, 3, 3, 1, 1, 0, 0), (1, 1, 4, 4, 1, 5, 3, 1, 1, 0, 0),
                (1, 1, 4, 4, 1, 3, 3, 0, 1, 0, 0), (1, 1, 4, 4, 1, 3, 3, 1, 1, -1, 0),
                (-1, 1, 4, 4, 1, 3, 3, 1, 1, 0, 0)]:
        gb = _native.Geom(*bad)
        st = lib.smmc_geom_check(ctypes.byref(gb), None, None)
        assert st == _native.SMMC_EGEOM
        with pytest.raises(GeometryError):
            _native.check(st)


def test_plans_and_workspace_without_gpu():
    g = ConvGeometry(512, 512, 7, 7, 3, 3, pad_h=1, pad_w=1)
    assert _native.plan_launches(g, 1, "exact") == 1
    assert _native.plan_launches(g, 1, "ffma") in (1, 2)
    assert _native.workspace_bytes(g, 1, "exact") == 0
    assert "split_k" in _native.plan_describe(g, 1)
    assert _native.plan_launches(g, 0) == 0


def test_tensor_core_plans_and_workspace_without_gpu():
    """The tensor-core split-K planner (host only): few-tile layers split
    their channel blocks and need a workspace, many-tile layers do not; the
    bf16x3 geometry plans over 3*c_i channels."""
    from paper_2411_15659_b200 import device
    small = ConvGeometry(512, 512, 7, 7, 3, 3, pad_h=1, pad_w=1)
    big = ConvGeometry(128, 128, 28, 28, 3, 3, pad_h=1, pad_w=1)
    assert device.tc_workspace_bytes(small, 1) > 0
    assert "split-K" in _native.tc_plan_describe(small, 1)
    assert device.tc_workspace_bytes(small, 1, split3=True) > 0
    assert "split-K" in device.tc3_plan_describe(small, 1)
    assert device.tc_workspace_bytes(big, 256) == 0
    assert device.tc_workspace_bytes(small, 0) == 0
    strided = ConvGeometry(16, 16, 16, 16, 3, 3, stride_h=2, stride_w=2, pad_h=1, pad_w=1)
    assert device.tc_workspace_bytes(strided, 4) == 0
    assert not device.tc_supported(strided)


def test_status_mapping():
    for st, exc in [(_native.SMMC_ESHAPE, smm.ShapeMismatchError),
                    (_native.SMMC_EUNSUPPORTED, smm.BackendUnsupportedError),
                    (_native.SMMC_ECUDA, DeviceError), (_native.SMMC_ENODEVICE, DeviceError),
                    (_native.SMMC_EINDEX, IndexError), (_native.SMMC_EWORKSPACE, ValueError)]:
        with pytest.raises(exc):
            _native.check(st)
    _native.check(0)
    with pytest.raises(smm.BackendUnsupportedError):
        _native.mode_id("tf32")


def test_compute_without_gpu_fails_loudly():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    g = ConvGeometry(2, 3, 6, 6, 3, 3)
    x = np.ones(g.input_shape, np.float32)
    w = np.ones(g.weights_smm_shape, np.float32)
    with pytest.raises(DeviceError):
        smm.smm_conv_single(x, w, g)
    lib = _native.lib()
    y = np.empty(g.output_shape, np.float32)
    gg = _native.Geom.of(g, 1)
    st = lib.smmc_conv2d_fwd_f32_host(x.ctypes.data, w.ctypes.data, y.ctypes.data,
                                      ctypes.byref(gg), 0, 0)
    assert st == _native.SMMC_ENODEVICE


def test_product_package_never_imports_the_oracle():
    pkg = Path(smm.__file__).resolve().parent
    for src in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = src.read_text()
        for needle in ("import oracle", "from oracle", "smm_oracle", "liboracle"):
            assert needle not in text, (src, needle)


def test_stem_plans_without_gpu():
    """c_i <= 4 3x3 s1 / 7x7 s2 / 11x11 s4 layers plan the direct stem kernel
    (one launch, no workspace); SMMC_STEM=0 and other kernels keep the tiled
    kernel."""
    import os
    for gt in [(3, 64, 224, 224, 3, 3, 1, 1, 1, 1), (3, 64, 224, 224, 7, 7, 2, 2, 3, 3),
               (3, 96, 227, 227, 11, 11, 4, 4, 0, 0), (1, 5, 13, 17, 3, 3, 2, 1, 1, 1)]:
        g = ConvGeometry(*gt)
        assert "direct stem" in _native.plan_describe(g, 8), gt
        assert _native.plan_launches(g, 8, "ffma") == 1
        assert _native.workspace_bytes(g, 8, "ffma") == 0
    for gt in [(3, 16, 20, 20, 5, 5, 1, 1, 2, 2), (5, 64, 40, 40, 7, 7, 2, 2, 3, 3)]:
        assert "direct stem" not in _native.plan_describe(ConvGeometry(*gt), 2), gt
    g = ConvGeometry(3, 64, 224, 224, 7, 7, 2, 2, 3, 3)
    os.environ["SMMC_STEM"] = "0"
    try:
        assert "direct stem" not in _native.plan_describe(g, 8)
    finally:
        del os.environ["SMMC_STEM"]
    # a single sample of a strided stem has too few tile blocks for the stem
    # kernel's long per-thread row loops: tiled split-K plans (SMMC_STEM=1 forces it)
    for gt in [(3, 64, 224, 224, 7, 7, 2, 2, 3, 3), (3, 96, 227, 227, 11, 11, 4, 4, 0, 0)]:
        g = ConvGeometry(*gt)
        assert "direct stem" not in _native.plan_describe(g, 1), gt
        os.environ["SMMC_STEM"] = "1"
        try:
            assert "direct stem" in _native.plan_describe(g, 1), gt
        finally:
            del os.environ["SMMC_STEM"]
    assert "direct stem" in _native.plan_describe(ConvGeometry(3, 64, 224, 224, 3, 3, 1, 1, 1, 1), 1)


def test_warp_tile_1x1_rule_without_gpu(monkeypatch):
    """1x1 layers with 32 < c_o <= 64 plan the warp-tile kernel where it measured
    faster (tools/narrow_n_probe.py): 2-12 warp tiles (16 px) per SM with the four
    schedulers >= 80 % evenly filled, or 2-3 tiles per SM; everything else keeps the
    tile kernels.  One launch, no workspace either way."""
    cases = [((256, 64, 56, 56, 1, 1), 8, True),     # config 3: 1568 tiles, 11 per SM
             ((256, 64, 56, 56, 1, 1), 2, True),     # 3 per SM
             ((256, 64, 56, 56, 1, 1), 4, False),    # 6 per SM: 2,2,1,1 warps per scheduler
             ((256, 64, 56, 56, 1, 1), 16, False),   # 22 per SM: second round of tiles
             ((256, 64, 28, 28, 1, 1), 2, False),    # 98 tiles: fewer than 2 per SM
             ((128, 64, 28, 28, 1, 1), 32, True),    # 11 per SM
             ((64, 256, 56, 56, 1, 1), 8, False),    # c_o > 64
             ((64, 32, 56, 56, 1, 1), 8, False),     # c_o <= 32
             ((512, 64, 56, 56, 1, 1), 8, False),    # weights exceed the resident budget
             ((80, 64, 56, 56, 1, 1), 8, True)]
    for gt, n, want in cases:
        g = ConvGeometry(*gt)
        desc = _native.plan_describe(g, n)
        assert ("warp-tile" in desc) == want, (gt, n, desc)
        assert "persistent 1x1" in desc
        assert _native.plan_launches(g, n, "ffma") == 1
        assert _native.workspace_bytes(g, n, "ffma") == 0
    g = ConvGeometry(256, 64, 56, 56, 1, 1)
    monkeypatch.setenv("SMMC_1X1_NARROW", "0")
    assert "warp-tile" not in _native.plan_describe(g, 8)
    monkeypatch.setenv("SMMC_1X1_NARROW", "2")
    assert "warp-tile" in _native.plan_describe(g, 16)


def test_one_wave_and_narrow_channel_plans_without_gpu(monkeypatch):
    """Planner rules for the reference harness's batch-1 layers (no GPU needed:
    plans are host logic): a one-wave split problem runs split-K reduced in the
    kernel on about one CTA per SM; a layer whose classic plan already fills the
    GPU keeps it; tap-major layers with c_o (mod 64) <= 32 use the 128 x 32
    tile; BASELINE shapes keep their measured plans."""
    alex3 = ConvGeometry(192, 384, 13, 13, 3, 3, 1, 1, 1, 1)
    d = _native.plan_describe(alex3, 1)
    assert "reduce=in-kernel" in d and "warp groups" in d, d
    ws_rule = _native.workspace_bytes(alex3, 1, "ffma")
    monkeypatch.setenv("SMMC_NO_SMALL_RULE", "1")
    d0 = _native.plan_describe(alex3, 1)
    assert "warp groups" not in d0 and "tile 128x128" in d0, d0   # the cost model's classic grid
    assert _native.workspace_bytes(alex3, 1, "ffma") != ws_rule
    monkeypatch.delenv("SMMC_NO_SMALL_RULE")
    # a classic grid that already fills one wave keeps its tile and splits; its
    # reduction moves into the kernel when the whole grid is co-resident
    vgg4 = ConvGeometry(256, 512, 28, 28, 3, 3, 1, 1, 1, 1)
    d4 = _native.plan_describe(vgg4, 1)
    assert "tile 64x128" in d4 and "split_k=11" in d4 and "reduce=in-kernel" in d4, d4
    assert _native.plan_launches(vgg4, 1, "ffma") == 1
    monkeypatch.setenv("SMMC_NO_INKERNEL_RULE", "1")
    assert "reduce=kernel" in _native.plan_describe(vgg4, 1)
    assert _native.plan_launches(vgg4, 1, "ffma") == 2
    monkeypatch.delenv("SMMC_NO_INKERNEL_RULE")
    # the paper's sweeps: c_o = 32 (layers.py:114-135)
    sweep = ConvGeometry(64, 32, 512, 512, 3, 3)
    assert "tile 128x32" in _native.plan_describe(sweep, 1)
    monkeypatch.setenv("SMMC_NO_BN32", "1")
    assert "tile 128x32" not in _native.plan_describe(sweep, 1)
    monkeypatch.delenv("SMMC_NO_BN32")
    assert "tile 128x32" not in _native.plan_describe(ConvGeometry(64, 64, 224, 224, 3, 3, 1, 1, 1, 1), 64)
    assert "tile 128x32" not in _native.plan_describe(ConvGeometry(3, 32, 64, 64, 5, 5), 1)  # generic K order
    # BASELINE config 1 / config 5 keep their table plans
    assert "tile 64x64" in _native.plan_describe(ConvGeometry(64, 64, 56, 56, 3, 3, 1, 1, 1, 1), 1)
    assert "tile 64x128" in _native.plan_describe(ConvGeometry(512, 512, 7, 7, 3, 3, 1, 1, 1, 1), 8)
