"""Drop-in replacement for the reference's SMM backend (``pkg/src/smmconv/smm.py``).

Same names, signatures, argument meaning and error behaviour; the compute runs
in the sm_100a kernels behind the C ABI (``include/smmc.h``).  Host (numpy)
callers get numpy results back (H2D + kernel + D2H per call, synchronous);
device-resident callers should use :mod:`.device` instead, which is
stream-ordered and never synchronises.

Kernel modes (keyword-only ``mode=`` on the conv drivers):
  * ``"ffma"`` (default, the product): register-tiled FFMA kernel;
    ``max|y - smm_ref| <= 1e-4 * max|smm_ref|`` (typically ~1e-6).
  * ``"exact"``: bitwise equal to the reference's ``smm_conv_single`` —
    (c, j, k) update order, separately rounded multiply and add.
Both are deterministic run to run, so ``smm_conv_parallel`` is bitwise equal
to ``smm_conv_single`` for every ``threads`` value, as in the reference
(``smm.py:254-260``).
"""

import ctypes

import numpy as np

from . import _native
from .errors import ShapeMismatchError
from .validation import (check_batch, check_input, check_weights,
                         check_weights_smm)

__all__ = [
    "repack_weights",
    "unpack_weights",
    "extract_slice",
    "shifted_view",
    "scalar_matrix_fma",
    "smm_conv_single",
    "smm_conv_parallel",
    "smm_conv_batched",
    "smm_workspace_elements",
    "gpu_workspace_bytes",
]


def _ptr(arr):
    return ctypes.c_void_p(arr.ctypes.data)


def repack_weights(weights, geom):
    """(out_ch, in_ch, k_h, k_w) -> (in_ch, k_w, k_h, out_ch) — smm.py:164-167.

    Host-side layout permutation done once per layer outside the timed path,
    as in the reference (runner.py:120-121).
    """
    check_weights(weights, geom)
    return np.ascontiguousarray(weights.transpose(1, 3, 2, 0))


def unpack_weights(weights_smm, geom):
    """Inverse of :func:`repack_weights` — smm.py:170-173."""
    check_weights_smm(weights_smm, geom)
    return np.ascontiguousarray(weights_smm.transpose(3, 0, 2, 1))


def smm_workspace_elements(geom, threads=1):
    """The reference's CPU scratch formula ``threads * padded_h * out_w``
    (smm.py:176-180).  The GPU kernels keep the slice in shared memory; their
    global scratch is :func:`gpu_workspace_bytes` (0 unless split-K)."""
    if threads < 1:
        raise ValueError("threads must be >= 1")
    return threads * geom.padded_h * geom.out_w


def gpu_workspace_bytes(geom, batch=1, mode="ffma"):
    """Global-memory scratch the GPU path needs for ``batch`` samples."""
    return _native.workspace_bytes(geom, batch, mode)


def extract_slice(inp, geom, c, j, buf):
    """Fill ``buf`` with the zero-packed slice for channel ``c``, kernel
    column ``j`` — smm.py:190-203, computed by a device kernel."""
    if not 0 <= c < geom.in_channels:
        raise IndexError(f"channel {c} out of range [0, {geom.in_channels})")
    if not 0 <= j < geom.k_w:
        raise IndexError(f"kernel column {j} out of range [0, {geom.k_w})")
    if (not isinstance(buf, np.ndarray) or buf.shape != (geom.padded_h, geom.out_w)
            or buf.dtype != np.float32 or not buf.flags.c_contiguous):
        raise ShapeMismatchError(
            f"slice buffer must be float32 {(geom.padded_h, geom.out_w)}")
    check_input(inp, geom)
    g = _native.Geom.of(geom, 1)
    _native.check(_native.lib().smmc_extract_slice_f32_host(
        _ptr(inp), ctypes.byref(g), c, j, _ptr(buf), _device()),
        "extract_slice")
    return buf


def shifted_view(buf, k, geom):
    """Rows ``k, k+s_h, ...`` of the slice buffer: a zero-copy numpy view
    (smm.py:206-214).  On the GPU this shift is loader index arithmetic."""
    if not 0 <= k < geom.k_h:
        raise IndexError(f"kernel row {k} out of range [0, {geom.k_h})")
    return buf[k:k + geom.out_h * geom.stride_h:geom.stride_h, :]


def scalar_matrix_fma(alpha, src, dst):
    """``dst += alpha * src`` (one rounded multiply, one rounded add per
    element) over equal-shaped 2-D views — smm.py:217-223, on the device."""
    if (not isinstance(src, np.ndarray) or not isinstance(dst, np.ndarray)
            or src.shape != dst.shape or src.ndim != 2):
        raise ShapeMismatchError(
            f"fma views must be equal-shaped 2-D: "
            f"{getattr(src, 'shape', None)} vs {getattr(dst, 'shape', None)}")
    if src.dtype != np.float32 or dst.dtype != np.float32:
        raise ShapeMismatchError("fma views must be float32")
    rows, cols = dst.shape
    if rows == 0 or cols == 0:
        return dst
    s = src if src.strides[1] == 4 else np.ascontiguousarray(src)
    d = dst if (dst.strides[1] == 4 and dst.strides[0] % 4 == 0
                and dst.strides[0] >= 0) else np.ascontiguousarray(dst)
    if s.strides[0] % 4 or s.strides[0] < 0:
        s = np.ascontiguousarray(s)
    _native.check(_native.lib().smmc_scalar_matrix_fma_f32_host(
        ctypes.c_float(np.float32(alpha)), _ptr(s), s.strides[0] // 4,
        _ptr(d), d.strides[0] // 4, rows, cols, _device()), "scalar_matrix_fma")
    if d is not dst:
        dst[...] = d
    return dst


def _device():
    # The host entry points stage on the caller's current torch device when
    # torch is imported; otherwise device 0.
    import sys
    torch = sys.modules.get("torch")
    if torch is not None:
        try:
            if torch.cuda.is_available():
                return torch.cuda.current_device()
        except Exception:  # pragma: no cover - torch without CUDA
            pass
    return 0


def _conv_host(x, weights_smm, geom, batch, mode):
    out_shape = (batch,) + geom.output_shape
    out = np.empty(out_shape, dtype=np.float32)
    g = _native.Geom.of(geom, batch)
    _native.check(_native.lib().smmc_conv2d_fwd_f32_host(
        _ptr(x), _ptr(weights_smm), _ptr(out), ctypes.byref(g),
        _native.mode_id(mode), _device()), "smm_conv")
    return out


def smm_conv_single(inp, weights_smm, geom, fused=True, *, mode="ffma"):
    """One sample ``(c_i, h, w)`` -> fresh ``(c_o, h', w')`` — smm.py:226-251.

    ``fused`` is accepted for signature parity; both settings run the same
    fused kernel (the reference's two settings are bitwise equal too,
    test_smm.py:206-214).
    """
    check_input(inp, geom)
    check_weights_smm(weights_smm, geom)
    return _conv_host(inp, weights_smm, geom, 1, mode)[0]


def smm_conv_parallel(inp, weights_smm, geom, threads, *, mode="ffma"):
    """Algorithm 2 entry (smm.py:254-306).  ``threads`` is validated like the
    reference (``< 1`` raises ValueError) but parallelism is the GPU's; the
    result is bitwise equal to :func:`smm_conv_single` for every value."""
    check_input(inp, geom)
    check_weights_smm(weights_smm, geom)
    if threads < 1:
        raise ValueError("threads must be >= 1")
    return _conv_host(inp, weights_smm, geom, 1, mode)[0]


def smm_conv_batched(x, weights_smm, geom, *, mode="ffma"):
    """``(N, c_i, h, w)`` -> ``(N, c_o, h', w')`` in ONE launch — the batched
    form of Conv2D.transform's per-sample loop (estimator.py:123-124)."""
    check_batch(x, geom)
    check_weights_smm(weights_smm, geom)
    return _conv_host(x, weights_smm, geom, x.shape[0], mode)
