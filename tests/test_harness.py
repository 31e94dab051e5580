"""layer configs, sweeps, CSV contract (CPU) and the GPU
benchmark runner with checksum cross-validation and scratch accounting."""

from pathlib import Path

import numpy as np
import pytest

from paper_2411_15659_b200 import ConfigError, ConvGeometry
from paper_2411_15659_b200 import harness as H

REF_PRESETS = Path("/root/reference/pkg/src/smmconv/presets")


def test_layer_config_parse_and_errors():
    specs = H.parse_layer_config(
        "# comment\n\nlayer name=a ci=3 co=8 h=32 w=30 kh=3 kw=5 ph=1  # tail\n"
        "layer name=b ci=4 co=4 h=9 w=9 kh=1 kw=1 sh=2 sw=2\n")
    assert [s.name for s in specs] == ["a", "b"]
    assert specs[0].geometry == ConvGeometry(3, 8, 32, 30, 3, 5, pad_h=1)
    assert specs[1].geometry.stride_w == 2 and specs[1].geometry.pad_w == 0
    for bad in ["lay name=a ci=1 co=1 h=4 w=4 kh=1 kw=1",
                "layer ci=1 co=1 h=4 w=4 kh=1 kw=1",
                "layer name=a ci=1 co=1 h=4 w=4 kh=1",
                "layer name=a ci=1 co=1 h=4 w=4 kh=1 kw=1 zz=3",
                "layer name=a ci=x co=1 h=4 w=4 kh=1 kw=1",
                "layer name=a ci=0 co=1 h=4 w=4 kh=1 kw=1",
                "layer name=a ci=1 ci=1 co=1 h=4 w=4 kh=1 kw=1",
                "layer name=a ci=1 co=1 h=4 w=4 kh=7 kw=1",
                "layer name=a ci=1 co=1 h=4 w=4 kh=1 kw= "]:
        with pytest.raises(ConfigError):
            H.parse_layer_config(bad)
    assert H.parse_layer_config("# nothing\n") == []


def test_sweeps_and_network():
    sizes = {k: len(H.sweep(k)) for k in H.SWEEP_KINDS}
    assert sizes == {"in_channels": 12, "spatial": 15, "kernel": 14, "out_channels": 6}
    vgg = H.builtin_network("vgg16")
    assert len(vgg) == 13 and vgg[0].name == "conv1_1"
    assert vgg[1].geometry == ConvGeometry(64, 64, 224, 224, 3, 3, pad_h=1, pad_w=1)
    with pytest.raises(ConfigError):
        H.sweep("nope")
    with pytest.raises(ConfigError):
        H.builtin_network("resnet")


@pytest.mark.skipif(not REF_PRESETS.exists(), reason="reference presets not mounted")
def test_reference_preset_files_parse():
    vgg = H.load_layer_config(REF_PRESETS / "vgg16.cfg")
    assert [s.geometry for s in vgg] == [s.geometry for s in H.builtin_network("vgg16")]
    assert len(H.load_layer_config(REF_PRESETS / "alexnet.cfg")) == 5
    assert len(H.load_layer_config(REF_PRESETS / "yolov3.cfg")) == 13


def test_csv_roundtrip_byte_identical():
    recs = [H.BenchRecord("conv1", "b200_smm", 148, 5, 0.000123456, 0, 3.25, 1234.5678),
            H.BenchRecord("conv1", "b200_bf16_tc", 148, 5, None, 0, None, None)]
    text = H.emit_csv(recs)
    assert text.splitlines()[0] == H.CSV_HEADER
    assert text.splitlines()[1] == "conv1,b200_smm,148,5,0.000123,0,3.2500,1234.5678"
    assert text.splitlines()[2] == "conv1,b200_bf16_tc,148,5,,0,,"
    assert H.emit_csv(H.parse_csv(text)) == text
    with pytest.raises(ConfigError):
        H.parse_csv("bad header\n")
    with pytest.raises(ConfigError):
        H.parse_csv(H.CSV_HEADER + "\na,b,1\n")
    with pytest.raises(ValueError):
        H.emit_csv([])


def test_run_bench_argument_errors():
    with pytest.raises(ValueError):
        H.run_bench([], ["b200_smm"], repeats=2)
    with pytest.raises(ValueError):
        H.run_bench([], ["cpu_smm"])


@pytest.mark.gpu
def test_run_bench_gpu_all_backends():
    specs = H.parse_layer_config(
        "layer name=l1 ci=64 co=64 h=28 w=28 kh=3 kw=3 ph=1 pw=1\n"
        "layer name=l2 ci=3 co=16 h=40 w=40 kh=7 kw=7 sh=2 sw=2 ph=3 pw=3\n"
        "layer name=l3 ci=32 co=32 h=16 w=16 kh=1 kw=1\n")
    recs = H.run_bench(specs, list(H.BACKENDS), repeats=3, batch=2)
    assert len(recs) == 3 * len(H.BACKENDS)
    by = {(r.layer, r.backend): r for r in recs}
    # strided stem: the bf16 tensor-core variant is unsupported, recorded as such
    assert by[("l2", "b200_bf16_tc")].unsupported
    assert by[("l2", "b200_bf16x3_tc")].unsupported
    for layer in ("l1", "l3"):  # fp32-accurate split-bf16: the fp32 checksum bar
        r, base = by[(layer, "b200_bf16x3_tc")], by[(layer, "b200_im2col")]
        assert abs(r.checksum - base.checksum) <= 1e-3 * abs(base.checksum)
        assert r.scratch_bytes > 0
    for layer in ("l1", "l2", "l3"):
        im2col = by[(layer, "b200_im2col")]
        g = next(s.geometry for s in specs if s.name == layer)
        assert im2col.scratch_bytes == 2 * g.in_channels * g.k_h * g.k_w * g.out_h * g.out_w * 4
        assert im2col.speedup_vs_im2col == pytest.approx(1.0)
        assert by[(layer, "b200_exact")].scratch_bytes == 0
        for b in ("b200_smm", "b200_exact"):
            r = by[(layer, b)]
            assert r.median_time_s > 0 and r.speedup_vs_im2col > 0
            assert abs(r.checksum - im2col.checksum) <= 1e-3 * abs(im2col.checksum)
    text = H.emit_csv(recs)
    assert H.emit_csv(H.parse_csv(text)) == text
