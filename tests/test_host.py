"""Host-side logic of the drop-in surface (no GPU needed): geometry,
validation, weight repacking, workspace formulas, estimator parameters.
Restates the reference's own unit tests for these pieces
(test_geometry.py, test_smm.py:19-47, 287-300, test_estimator.py)."""

import numpy as np
import pytest
from hypothesis import given, strategies as st

import paper_2411_15659_b200 as smm
from conftest import sample_geometry
from paper_2411_15659_b200 import (BackendUnsupportedError, ConvGeometry,
                                   GeometryError, ShapeMismatchError, output_shape)


def test_output_shapes():
    assert output_shape(ConvGeometry(1, 1, 4, 4, 3, 3)) == (2, 2)
    assert output_shape(ConvGeometry(1, 1, 5, 5, 1, 1)) == (5, 5)
    assert output_shape(ConvGeometry(3, 64, 224, 224, 11, 11, stride_h=4, stride_w=4,
                                     pad_h=2, pad_w=2)) == (55, 55)
    g = ConvGeometry(1, 1, 10, 6, 5, 3, stride_h=2, stride_w=1, pad_h=0, pad_w=1)
    assert (g.out_h, g.out_w, g.padded_h, g.padded_w) == (3, 6, 10, 8)


@pytest.mark.parametrize("bad", [dict(in_channels=0), dict(out_channels=0), dict(in_h=0),
                                 dict(k_w=0), dict(stride_h=0), dict(pad_h=-1)])
def test_rejects_nonpositive(bad):
    kw = dict(in_channels=1, out_channels=1, in_h=4, in_w=4, k_h=3, k_w=3)
    kw.update(bad)
    with pytest.raises(GeometryError):
        ConvGeometry(**kw)


def test_rejects_kernel_and_empty_output_and_non_int():
    with pytest.raises(GeometryError):
        ConvGeometry(1, 1, 4, 4, 5, 3)
    ConvGeometry(1, 1, 4, 4, 5, 3, pad_h=1)
    with pytest.raises(GeometryError):
        ConvGeometry(1, 1, 4, 4, 3, 7, pad_h=0, pad_w=1)
    with pytest.raises(GeometryError):
        ConvGeometry(1.0, 1, 4, 4, 3, 3)
    with pytest.raises(GeometryError):
        ConvGeometry(True, 1, 4, 4, 3, 3)
    assert issubclass(GeometryError, ValueError)


@given(k=st.integers(1, 6), p=st.integers(0, 3))
def test_output_monotone(k, p):
    base = ConvGeometry(1, 1, 8, 8, k, k, pad_h=p, pad_w=p)
    more_pad = ConvGeometry(1, 1, 8, 8, k, k, pad_h=p + 1, pad_w=p + 1)
    assert more_pad.out_h >= base.out_h and more_pad.out_w >= base.out_w


def test_layout_shapes_and_flops():
    g = ConvGeometry(64, 64, 56, 56, 3, 3, pad_h=1, pad_w=1)
    assert g.weights_shape == (64, 64, 3, 3)
    assert g.weights_smm_shape == (64, 3, 3, 64)
    assert g.flops(1) == 2 * 64 * 56 * 56 * 64 * 9
    assert g.compulsory_bytes(1) == 4 * (64 * 56 * 56 * 2 + 64 * 64 * 9)
    assert g.as_abi(5) == (5, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1)


def test_repack_roundtrip_and_index_formula(rng):
    for i in range(50):
        g = sample_geometry(rng)
        w = smm.random_tensor(g.weights_shape, i)
        ws = smm.repack_weights(w, g)
        assert ws.shape == g.weights_smm_shape
        assert np.array_equal(smm.unpack_weights(ws, g), w)
    g = ConvGeometry(2, 3, 6, 6, 3, 3)
    w = smm.random_tensor(g.weights_shape, 9)
    ws = smm.repack_weights(w, g)
    for m, c, k, j in [(0, 0, 0, 0), (2, 1, 2, 1), (1, 0, 1, 2)]:
        assert ws[c, j, k, m] == w[m, c, k, j]
    single = ConvGeometry(1, 1, 3, 3, 1, 1)
    assert smm.repack_weights(np.array([[[[2.5]]]], np.float32), single)[0, 0, 0, 0] == 2.5


def test_validation_errors():
    g = ConvGeometry(2, 3, 6, 6, 3, 3)
    with pytest.raises(ShapeMismatchError):
        smm.repack_weights(np.zeros(g.weights_smm_shape, np.float32), g)
    with pytest.raises(ShapeMismatchError):
        smm.repack_weights(np.zeros(g.weights_shape, np.float64), g)
    with pytest.raises(ShapeMismatchError):
        smm.unpack_weights([[1.0]], g)
    # validation happens before any device work, so it also holds on CPU boxes
    x = np.zeros(g.input_shape, np.float32)
    with pytest.raises(ShapeMismatchError):
        smm.smm_conv_single(x, np.zeros(g.weights_shape, np.float32), g)
    with pytest.raises(ShapeMismatchError):
        smm.smm_conv_parallel(x[:1], np.zeros(g.weights_smm_shape, np.float32), g, 2)
    with pytest.raises(ShapeMismatchError):
        smm.scalar_matrix_fma(1.0, np.zeros((2, 3), np.float32), np.zeros((3, 2), np.float32))
    with pytest.raises(IndexError):
        smm.extract_slice(x, g, 2, 0, np.empty((g.padded_h, g.out_w), np.float32))
    with pytest.raises(IndexError):
        smm.extract_slice(x, g, 0, 3, np.empty((g.padded_h, g.out_w), np.float32))
    with pytest.raises(ShapeMismatchError):
        smm.extract_slice(x, g, 0, 0, np.empty((4, 3), np.float32))
    with pytest.raises(IndexError):
        smm.shifted_view(np.empty((g.padded_h, g.out_w), np.float32), 3, g)


def test_shifted_view_zero_copy():
    g = ConvGeometry(1, 1, 7, 5, 3, 3, stride_h=3)
    buf = np.arange(g.padded_h * g.out_w, dtype=np.float32).reshape(g.padded_h, g.out_w)
    for k in range(3):
        v = smm.shifted_view(buf, k, g)
        assert v.shape == (g.out_h, g.out_w)
        assert np.shares_memory(v, buf)
        assert np.array_equal(v, buf[[k + 3 * r for r in range(g.out_h)]])


def test_workspace_formulas():
    g = ConvGeometry(1, 1, 64, 64, 3, 3)
    assert smm.smm_workspace_elements(g, 1) == 64 * 62 == 3968
    assert smm.smm_workspace_elements(ConvGeometry(1, 1, 64, 64, 3, 3, pad_h=1), 1) == 4092
    assert smm.smm_workspace_elements(g, 8) == 8 * 3968
    with pytest.raises(ValueError):
        smm.smm_workspace_elements(g, 0)


def test_estimator_params_and_fit_without_gpu():
    from sklearn.base import clone
    from sklearn.exceptions import NotFittedError
    est = smm.Conv2D(out_channels=5, kernel_size=(3, 1), stride=2, padding=(1, 0),
                     threads=2, seed=9)
    params = est.get_params()
    assert params["out_channels"] == 5 and params["kernel_size"] == (3, 1)
    assert clone(est).get_params() == params
    with pytest.raises(NotFittedError):
        smm.Conv2D().transform(smm.random_tensor((1, 2, 8, 8), 0))
    X = smm.random_tensor((3, 2, 8, 8), 0)
    a = smm.Conv2D(out_channels=2, seed=3).fit(X)
    b = smm.Conv2D(out_channels=2, seed=3).fit(X)
    assert np.array_equal(a.weights_, b.weights_)
    assert np.array_equal(a.weights_, smm.random_tensor((2, 2, 3, 3), 3))
    assert a.weights_smm_.shape == (2, 3, 3, 2)
    with pytest.raises(ValueError):
        smm.Conv2D(out_channels=2).fit(np.zeros((4, 4), np.float32))
    with pytest.raises(ValueError):
        smm.Conv2D(out_channels=2).fit(np.full((1, 1, 4, 4), np.nan, np.float32))
    with pytest.raises(ValueError):
        smm.Conv2D(out_channels=2, backend="winograd").fit(X)
    with pytest.raises(BackendUnsupportedError):
        smm.Conv2D(out_channels=2, backend="im2col").fit(X)
    # the split-bf16 tensor-core backend: c_i % 8 == 0 and stride 1 (host check at fit)
    with pytest.raises(BackendUnsupportedError):
        smm.Conv2D(out_channels=2, backend="smm_tc3").fit(X)
    X8 = np.zeros((1, 8, 6, 6), np.float32)
    assert smm.Conv2D(out_channels=2, backend="smm_tc3").fit(X8).geometry_.in_channels == 8
    with pytest.raises(BackendUnsupportedError):
        smm.Conv2D(out_channels=2, stride=2, backend="smm_tc3").fit(X8)
    with pytest.raises(ValueError):
        smm.Conv2D(out_channels=2, weights=np.zeros((1, 2, 3, 3), np.float32)).fit(X)


def test_estimator_threads_is_advisory_like_the_reference():
    """The reference's Conv2D never validates `threads` (estimator.py:99-110
    only branches on threads > 1): numpy ints and values < 1 fit fine."""
    X = smm.random_tensor((1, 2, 6, 6), 0)
    for t in (np.int64(4), np.int32(1), 0, -3, 16):
        assert smm.Conv2D(out_channels=2, threads=t).fit(X).geometry_.out_h == 4
    with pytest.raises(ValueError):
        smm.Conv2D(out_channels=2, threads="4").fit(X)
