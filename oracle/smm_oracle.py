"""ORACLE — TEST INFRASTRUCTURE ONLY (the checker, never the product).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` leg may import this module.  The product package
(``paper_2411_15659_b200``) never imports it and has no CPU compute path.

Two restatements of the reference's SMM-Conv CPU algorithm
(/root/reference/pkg/src/smmconv/smm.py), both bit-exact with
``smm_conv_single`` (pinned by tests/test_oracle.py against the golden
vectors the reference itself produced, tests/golden/make_golden.py):

* ``smm_conv_np`` — numpy, one vectorised update per (c, j, k) tap over all
  output channels: ``out += w[c,j,k,:,None,None] * window`` (float32 multiply,
  then float32 add: the same two roundings as smm.py:76-81 / 100-114).
* ``smm_conv_c`` — the C restatement (oracle/smm_oracle.c) incl. the
  Algorithm 2 thread-parallel driver (smm.py:254-306); fast enough to be the
  CPU baseline.

Parity metrics: ``max_abs_ratio`` = max|y - ref| / max|ref| in float64 (the
BASELINE.json bar, 1e-4 fp32 / 2e-2 bf16) and ``max_rel_diff`` (the
reference's elementwise metric, tensors.py:65-78).
"""

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "build" / "liboracle_smm.so"

__all__ = ["smm_conv_np", "smm_conv_c", "conv_ref_c", "extract_slice_c",
           "max_abs_ratio", "max_rel_diff", "build_oracle", "repack"]


class _Geom(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in
                ("n", "c_i", "h", "w", "c_o", "k_h", "k_w", "s_h", "s_w",
                 "p_h", "p_w")]


def build_oracle(force=False):
    """Compile oracle/smm_oracle.c with the committed Makefile."""
    src = HERE / "smm_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build_oracle()
        lib = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        G = ctypes.POINTER(_Geom)
        lib.oracle_smm_conv.argtypes = [P, P, P, G, ctypes.c_int]
        lib.oracle_smm_conv.restype = ctypes.c_int
        lib.oracle_conv_ref.argtypes = [P, P, P, G]
        lib.oracle_conv_ref.restype = ctypes.c_int
        lib.oracle_extract_slice.argtypes = [P, G, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_extract_slice.restype = ctypes.c_int
        _lib = lib
    return _lib


def _geom_fields(geom):
    return dict(c_i=geom.in_channels, h=geom.in_h, w=geom.in_w,
                c_o=geom.out_channels, k_h=geom.k_h, k_w=geom.k_w,
                s_h=geom.stride_h, s_w=geom.stride_w, p_h=geom.pad_h,
                p_w=geom.pad_w)


def repack(w_oihw):
    """(c_o, c_i, k_h, k_w) -> (c_i, k_w, k_h, c_o) — smm.py:164-167."""
    return np.ascontiguousarray(w_oihw.transpose(1, 3, 2, 0))


def smm_conv_np(x, w_smm, geom):
    """numpy restatement of smm_conv_single (smm.py:226-251) for one sample
    (c_i, h, w) or a batch (n, c_i, h, w)."""
    if x.ndim == 4:
        return np.stack([smm_conv_np(xi, w_smm, geom) for xi in x])
    oh, ow = geom.out_h, geom.out_w
    out = np.zeros((geom.out_channels, oh, ow), dtype=np.float32)
    pad = np.zeros((geom.in_channels, geom.padded_h, geom.padded_w), np.float32)
    pad[:, geom.pad_h:geom.pad_h + geom.in_h, geom.pad_w:geom.pad_w + geom.in_w] = x
    sh, sw = geom.stride_h, geom.stride_w
    for c in range(geom.in_channels):
        for j in range(geom.k_w):
            buf = pad[c][:, j:j + ow * sw:sw]               # extract (smm.py:56-73)
            for k in range(geom.k_h):
                win = buf[k:k + oh * sh:sh, :]               # shifted view (206-214)
                wk = w_smm[c, j, k, :].astype(np.float32)
                prod = wk[:, None, None] * win[None, :, :]   # rounded multiply
                out += prod                                  # rounded add
    return out


def smm_conv_c(x, w_smm, geom, threads=1):
    """C restatement; x is (c_i,h,w) or (n,c_i,h,w); Algorithm 2 when threads>1."""
    lib = _load()
    single = x.ndim == 3
    xb = np.ascontiguousarray(x[None] if single else x, dtype=np.float32)
    w = np.ascontiguousarray(w_smm, dtype=np.float32)
    n = xb.shape[0]
    y = np.empty((n, geom.out_channels, geom.out_h, geom.out_w), np.float32)
    g = _Geom(n=n, **_geom_fields(geom))
    st = lib.oracle_smm_conv(xb.ctypes.data, w.ctypes.data, y.ctypes.data,
                             ctypes.byref(g), int(threads))
    if st:
        raise RuntimeError(f"oracle_smm_conv failed ({st})")
    return y[0] if single else y


def conv_ref_c(x, w_oihw, geom):
    """C restatement of conv_ref (reference.py:18-38), (c, k, j) order."""
    lib = _load()
    single = x.ndim == 3
    xb = np.ascontiguousarray(x[None] if single else x, dtype=np.float32)
    w = np.ascontiguousarray(w_oihw, dtype=np.float32)
    n = xb.shape[0]
    y = np.empty((n, geom.out_channels, geom.out_h, geom.out_w), np.float32)
    g = _Geom(n=n, **_geom_fields(geom))
    lib.oracle_conv_ref(xb.ctypes.data, w.ctypes.data, y.ctypes.data, ctypes.byref(g))
    return y[0] if single else y


def extract_slice_c(x, geom, c, j):
    lib = _load()
    xs = np.ascontiguousarray(x, dtype=np.float32)
    buf = np.empty((geom.padded_h, geom.out_w), np.float32)
    g = _Geom(n=1, **_geom_fields(geom))
    lib.oracle_extract_slice(xs.ctypes.data, ctypes.byref(g), int(c), int(j), buf.ctypes.data)
    return buf


def max_abs_ratio(y, ref):
    """max|y - ref| / max|ref| in float64 (BASELINE.json parity metric)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.shape != ref.shape:
        raise ValueError(f"shape mismatch {y.shape} vs {ref.shape}")
    if ref.size == 0:
        return 0.0
    scale = float(np.max(np.abs(ref)))
    err = float(np.max(np.abs(y - ref)))
    return err / scale if scale > 0 else err


def max_rel_diff(a, b):
    """Reference's elementwise metric (tensors.py:65-78)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.size == 0:
        return 0.0
    denom = np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-12)
    return float(np.max(np.abs(a.astype(np.float64) - b.astype(np.float64)) / denom))


def host_threads():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
