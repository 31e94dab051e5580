"""ctypes binding of the C ABI (``include/smmc.h``) exported by ``lib/libsmmc.so``.

The library is the only compute path: if it is missing or no GPU is visible
the calls raise ``DeviceError`` — nothing here (or anywhere in the package)
computes a convolution on the CPU.
"""

import ctypes
import os
import threading
from pathlib import Path

from .errors import (BackendUnsupportedError, DeviceError, GeometryError,
                     ShapeMismatchError, SmmConvError)

__all__ = ["lib", "Geom", "check", "LIB_PATH", "MODES", "mode_id",
           "EXPORTED_SYMBOLS"]

LIB_PATH = Path(os.environ.get(
    "SMMC_LIB", Path(__file__).resolve().parent / "lib" / "libsmmc.so"))

SMMC_OK = 0
SMMC_EGEOM = 1
SMMC_ESHAPE = 2
SMMC_EUNSUPPORTED = 3
SMMC_EWORKSPACE = 4
SMMC_ECUDA = 5
SMMC_ENODEVICE = 6
SMMC_EINDEX = 7

MODES = {"ffma": 0, "exact": 1}

# Every function include/smmc.h declares (tests/test_boundary.py checks the
# header and the shared object against this list).
EXPORTED_SYMBOLS = (
    "smmc_abi_version", "smmc_last_error", "smmc_geom_check",
    "smmc_workspace_bytes", "smmc_conv2d_fwd_f32", "smmc_conv2d_fwd_f32_host",
    "smmc_extract_slice_f32", "smmc_scalar_matrix_fma_f32",
    "smmc_extract_slice_f32_host", "smmc_scalar_matrix_fma_f32_host",
    "smmc_plan_launches", "smmc_plan_describe", "smmc_tc_plan_describe", "smmc_launch_count",
    "smmc_tc_supported", "smmc_pack_input_bf16_nhwc", "smmc_pack_weights_bf16",
    "smmc_conv2d_fwd_bf16_tc", "smmc_pack_input_bf16x3_nhwc", "smmc_pack_weights_bf16x3",
    "smmc_conv2d_fwd_bf16x3_tc", "smmc_tc_workspace_bytes", "smmc_conv2d_fwd_bf16_tc_ws",
    "smmc_im2col_bytes", "smmc_im2col_pack_f32",
    "smmc_conv2d_fwd_f32_gather", "smmc_gather_workspace_bytes", "smmc_ipc_handle",
    "smmc_ipc_open", "smmc_ipc_close", "smmc_host_alloc_pinned", "smmc_host_free_pinned",
    "smmc_layer_create", "smmc_layer_forward_host", "smmc_layer_destroy",
    "smmc_layer_forward_host_async", "smmc_layer_wait",
    "smmc_autotune_f32", "smmc_autotune_clear",
)

SMMC_MAX_OUT = 8
SMMC_IPC_HANDLE_BYTES = 64


class Geom(ctypes.Structure):
    """``smmc_geom``: n, c_i, h, w, c_o, k_h, k_w, s_h, s_w, p_h, p_w (int32)."""

    _fields_ = [(f, ctypes.c_int32) for f in
                ("n", "c_i", "h", "w", "c_o", "k_h", "k_w", "s_h", "s_w",
                 "p_h", "p_w")]

    @classmethod
    def of(cls, geom, batch=1):
        return cls(*geom.as_abi(batch))


def mode_id(mode):
    if isinstance(mode, int) and mode in MODES.values():
        return mode
    try:
        return MODES[mode]
    except (KeyError, TypeError):
        raise BackendUnsupportedError(
            f"unknown kernel mode {mode!r}; choose from {sorted(MODES)}") from None


_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_GP = ctypes.POINTER(Geom)

_SIGNATURES = {
    "smmc_abi_version": (ctypes.c_int, []),
    "smmc_last_error": (ctypes.c_char_p, []),
    "smmc_geom_check": (ctypes.c_int, [_GP, ctypes.POINTER(_I32), ctypes.POINTER(_I32)]),
    "smmc_workspace_bytes": (ctypes.c_size_t, [_GP, ctypes.c_int]),
    "smmc_conv2d_fwd_f32": (ctypes.c_int, [_P, _P, _P, _GP, ctypes.c_int, _P,
                                           ctypes.c_size_t, _P]),
    "smmc_conv2d_fwd_f32_host": (ctypes.c_int, [_P, _P, _P, _GP, ctypes.c_int,
                                                ctypes.c_int]),
    "smmc_extract_slice_f32": (ctypes.c_int, [_P, _GP, _I32, _I32, _P, _P]),
    "smmc_scalar_matrix_fma_f32": (ctypes.c_int, [ctypes.c_float, _P, _I64, _P,
                                                  _I64, _I32, _I32, _P]),
    "smmc_extract_slice_f32_host": (ctypes.c_int, [_P, _GP, _I32, _I32, _P,
                                                   ctypes.c_int]),
    "smmc_scalar_matrix_fma_f32_host": (ctypes.c_int, [ctypes.c_float, _P, _I64,
                                                       _P, _I64, _I32, _I32,
                                                       ctypes.c_int]),
    "smmc_plan_launches": (ctypes.c_int, [_GP, ctypes.c_int]),
    "smmc_plan_describe": (ctypes.c_int, [_GP, ctypes.c_int, ctypes.c_char_p,
                                          ctypes.c_size_t]),
    "smmc_launch_count": (ctypes.c_uint64, []),
    "smmc_autotune_f32": (ctypes.c_int, [_GP, ctypes.c_int, ctypes.c_char_p, ctypes.c_size_t]),
    "smmc_autotune_clear": (ctypes.c_int, []),
    "smmc_tc_plan_describe": (ctypes.c_int, [_GP, ctypes.c_char_p, ctypes.c_size_t]),
    "smmc_tc_supported": (ctypes.c_int, [_GP]),
    "smmc_pack_input_bf16_nhwc": (ctypes.c_int, [_P, _P, _GP, _P]),
    "smmc_pack_weights_bf16": (ctypes.c_int, [_P, _P, _GP, _P]),
    "smmc_conv2d_fwd_bf16_tc": (ctypes.c_int, [_P, _P, _P, _GP, _P]),
    "smmc_pack_input_bf16x3_nhwc": (ctypes.c_int, [_P, _P, _GP, _P]),
    "smmc_pack_weights_bf16x3": (ctypes.c_int, [_P, _P, _GP, _P]),
    "smmc_conv2d_fwd_bf16x3_tc": (ctypes.c_int, [_P, _P, _P, _GP, _P, ctypes.c_size_t, _P]),
    "smmc_tc_workspace_bytes": (ctypes.c_size_t, [_GP, ctypes.c_int]),
    "smmc_conv2d_fwd_bf16_tc_ws": (ctypes.c_int, [_P, _P, _P, _GP, _P, ctypes.c_size_t, _P]),
    "smmc_im2col_bytes": (ctypes.c_size_t, [_GP]),
    "smmc_im2col_pack_f32": (ctypes.c_int, [_P, _P, _GP, _P]),
    "smmc_conv2d_fwd_f32_gather": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_void_p),
                                                  ctypes.c_int, _GP, ctypes.c_int, ctypes.c_int,
                                                  _P, ctypes.c_size_t, _P]),
    "smmc_gather_workspace_bytes": (ctypes.c_size_t, [_GP]),
    "smmc_ipc_handle": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_size_t)]),
    "smmc_ipc_open": (ctypes.c_int, [_P, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "smmc_ipc_close": (ctypes.c_int, [_P, ctypes.c_size_t]),
    "smmc_host_alloc_pinned": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "smmc_host_free_pinned": (ctypes.c_int, [_P]),
    "smmc_layer_create": (ctypes.c_int, [_P, _GP, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]),
    "smmc_layer_forward_host": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int]),
    "smmc_layer_destroy": (ctypes.c_int, [_P]),
    "smmc_layer_forward_host_async": (ctypes.c_int, [_P, _P, _P, ctypes.c_int, ctypes.c_int]),
    "smmc_layer_wait": (ctypes.c_int, [_P]),
}


def lib():
    """Load (once) and return the native library, or raise DeviceError."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise DeviceError(
                    f"native library {LIB_PATH} is not built; run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            try:
                handle = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise DeviceError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in _SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error():
    msg = lib().smmc_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(status, what="smmc"):
    """Map a C status to the reference's exception types."""
    if status == SMMC_OK:
        return
    msg = f"{what}: {last_error()}"
    if status == SMMC_EGEOM:
        raise GeometryError(msg)
    if status == SMMC_ESHAPE:
        raise ShapeMismatchError(msg)
    if status == SMMC_EUNSUPPORTED:
        raise BackendUnsupportedError(msg)
    if status == SMMC_EWORKSPACE:
        raise ValueError(msg)
    if status == SMMC_EINDEX:
        raise IndexError(msg)
    if status in (SMMC_ECUDA, SMMC_ENODEVICE):
        raise DeviceError(msg)
    raise SmmConvError(f"{what}: status {status}: {last_error()}")


def launch_count():
    return int(lib().smmc_launch_count())


def plan_describe(geom, batch=1, mode="ffma"):
    buf = ctypes.create_string_buffer(256)
    g = Geom.of(geom, batch)
    check(lib().smmc_plan_describe(ctypes.byref(g), mode_id(mode), buf, 256),
          "smmc_plan_describe")
    return buf.value.decode()


def autotune(geom, batch=1, iters=10):
    """Measure the candidate kernel plans of (geom, batch) on the current device
    and keep the fastest for this process (smmc_autotune_f32); returns the
    library's one-line report.  Call before sizing workspaces for the shape."""
    buf = ctypes.create_string_buffer(256)
    g = Geom.of(geom, batch)
    check(lib().smmc_autotune_f32(ctypes.byref(g), int(iters), buf, 256), "smmc_autotune_f32")
    return buf.value.decode()


def autotune_clear():
    check(lib().smmc_autotune_clear(), "smmc_autotune_clear")


def autotune_enabled():
    """SMMC_AUTOTUNE=1 turns per-shape autotuning on wherever a layer is fitted
    (device.SmmConv2d, the estimator, the harness backends)."""
    return os.environ.get("SMMC_AUTOTUNE", "0") not in ("", "0")


def tc_plan_describe(geom, batch=1):
    buf = ctypes.create_string_buffer(256)
    g = Geom.of(geom, batch)
    check(lib().smmc_tc_plan_describe(ctypes.byref(g), buf, 256), "smmc_tc_plan_describe")
    return buf.value.decode()


def plan_launches(geom, batch=1, mode="ffma"):
    g = Geom.of(geom, batch)
    return int(lib().smmc_plan_launches(ctypes.byref(g), mode_id(mode)))


def gather_workspace_bytes(geom_local, batch=1):
    g = Geom.of(geom_local, batch)
    return int(lib().smmc_gather_workspace_bytes(ctypes.byref(g)))


def ipc_handle(dev_ptr):
    """(handle bytes, byte offset) of a device pointer, for smmc_ipc_open in a
    peer process."""
    buf = ctypes.create_string_buffer(SMMC_IPC_HANDLE_BYTES)
    off = ctypes.c_size_t(0)
    check(lib().smmc_ipc_handle(ctypes.c_void_p(dev_ptr), buf, ctypes.byref(off)),
          "smmc_ipc_handle")
    return buf.raw, int(off.value)


def ipc_open(handle, offset):
    """Map a peer's device pointer (from ipc_handle) into this process."""
    if len(handle) != SMMC_IPC_HANDLE_BYTES:
        raise ShapeMismatchError("IPC handle must be SMMC_IPC_HANDLE_BYTES bytes")
    ptr = ctypes.c_void_p(0)
    check(lib().smmc_ipc_open(ctypes.create_string_buffer(handle, SMMC_IPC_HANDLE_BYTES),
                              offset, ctypes.byref(ptr)), "smmc_ipc_open")
    return int(ptr.value)


def ipc_close(dev_ptr, offset):
    check(lib().smmc_ipc_close(ctypes.c_void_p(dev_ptr), offset), "smmc_ipc_close")


class Layer:
    """A fitted conv layer (smmc_layer): W_smm uploaded once to `device`;
    ``forward(x, y)`` runs the host-buffer pipeline on float32 C-contiguous
    numpy arrays (x: (n, c_i, h, w) -> y: (n, c_o, h', w'))."""

    def __init__(self, weights_smm, geom, device=0):
        import numpy as np
        w = np.ascontiguousarray(weights_smm, dtype=np.float32)
        if w.shape != geom.weights_smm_shape:
            raise ShapeMismatchError(
                f"weights_smm has shape {w.shape}, expected {geom.weights_smm_shape}")
        self.geom = geom
        self._h = ctypes.c_void_p(0)
        g = Geom.of(geom, 1)
        check(lib().smmc_layer_create(w.ctypes.data_as(ctypes.c_void_p), ctypes.byref(g),
                                      int(device), ctypes.byref(self._h)), "smmc_layer_create")

    def forward(self, x, y, mode="ffma"):
        n = int(x.shape[0])
        check(lib().smmc_layer_forward_host(self._h, ctypes.c_void_p(x.ctypes.data),
                                            ctypes.c_void_p(y.ctypes.data), n, mode_id(mode)),
              "smmc_layer_forward_host")
        return y

    def forward_async(self, x, y, mode="ffma"):
        """Enqueue x -> y on the layer's own staging buffers and streams and
        return; ``x`` and ``y`` must stay alive (and ``y`` unread) until
        ``wait()``.  Calls on different layers overlap their copies."""
        n = int(x.shape[0])
        check(lib().smmc_layer_forward_host_async(self._h, ctypes.c_void_p(x.ctypes.data),
                                                  ctypes.c_void_p(y.ctypes.data), n,
                                                  mode_id(mode)), "smmc_layer_forward_host_async")
        return y

    def wait(self):
        check(lib().smmc_layer_wait(self._h), "smmc_layer_wait")

    def close(self):
        if self._h and self._h.value:
            lib().smmc_layer_destroy(self._h)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def pinned_empty(shape, dtype="float32"):
    """A numpy array in page-locked host memory (smmc_host_alloc_pinned),
    freed when the array is garbage-collected."""
    import weakref

    import numpy as np
    dt = np.dtype(dtype)
    count = 1
    for d in shape:
        count *= int(d)
    nbytes = max(count * dt.itemsize, 1)
    ptr = ctypes.c_void_p(0)
    check(lib().smmc_host_alloc_pinned(nbytes, ctypes.byref(ptr)), "smmc_host_alloc_pinned")
    buf = (ctypes.c_char * nbytes).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=count).reshape(shape)
    weakref.finalize(buf, lib().smmc_host_free_pinned, ctypes.c_void_p(ptr.value))
    return arr


def pinned_copy(a):
    """Page-locked copy of a numpy array."""
    import numpy as np
    a = np.ascontiguousarray(a)
    out = pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def workspace_bytes(geom, batch=1, mode="ffma"):
    g = Geom.of(geom, batch)
    return int(lib().smmc_workspace_bytes(ctypes.byref(g), mode_id(mode)))
