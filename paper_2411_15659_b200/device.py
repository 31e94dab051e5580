"""Device-resident entry points over torch CUDA tensors.

PyTorch is plumbing here (device memory, streams); the compute is the C ABI's
``smmc_conv2d_fwd_f32`` launched on torch's current stream, with no host
synchronisation — usable inside CUDA-graph capture.
"""

import ctypes

from . import _native
from .errors import DeviceError, ShapeMismatchError

__all__ = ["conv2d", "conv2d_gather", "repack_weights", "SmmConv2d"]


def _torch():
    import torch
    return torch


def _check_tensor(t, shape, name, align=16):
    torch = _torch()
    if not isinstance(t, torch.Tensor):
        raise ShapeMismatchError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ShapeMismatchError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != torch.float32:
        raise ShapeMismatchError(f"{name} must be float32, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ShapeMismatchError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if not t.is_contiguous():
        raise ShapeMismatchError(f"{name} must be contiguous")
    if t.data_ptr() % align:
        raise ShapeMismatchError(f"{name} must be {align}-byte aligned")
    return t


def repack_weights(weights, geom):
    """OIHW -> (c_i, k_w, k_h, c_o) on the device (once per layer, untimed)."""
    _check_tensor(weights, geom.weights_shape, "weight tensor")
    return weights.permute(1, 3, 2, 0).contiguous()


def new_workspace(geom, batch, mode="ffma", device=None):
    """A zero-filled workspace for ``conv2d`` of this problem (None if the plan
    needs none)."""
    torch = _torch()
    need = _native.workspace_bytes(geom, batch, mode)
    if not need:
        return None
    return torch.zeros(need, dtype=torch.uint8, device=device or torch.cuda.current_device())


def conv2d(x, weights_smm, geom, *, mode="ffma", out=None, workspace=None):
    """Batched NCHW forward conv on torch's current stream.

    ``x`` (N, c_i, h, w), ``weights_smm`` (c_i, k_w, k_h, c_o) on the same
    device; returns ``out`` (N, c_o, h', w').  Split-K problems need a
    workspace: pass one (uint8 tensor of ``_native.workspace_bytes`` bytes,
    e.g. ``new_workspace``) to stay allocation-free, else a zeroed one is
    taken from torch's caching allocator.  A workspace must be ZERO-FILLED
    before its first use (its leading counter region is zero at rest: every
    launch that uses split-K counters re-arms them), and may then be reused
    by any sequence of layers on one stream.
    """
    torch = _torch()
    if not isinstance(x, torch.Tensor) or x.dim() != 4:
        raise ShapeMismatchError("x must be a 4-D torch.Tensor (N, c_i, h, w)")
    n = x.shape[0]
    _check_tensor(x, (n,) + geom.input_shape, "input batch", align=4)
    _check_tensor(weights_smm, geom.weights_smm_shape, "repacked weight tensor")
    if weights_smm.device != x.device:
        raise ShapeMismatchError("x and weights_smm must be on the same device")
    if out is None:
        out = torch.empty((n,) + geom.output_shape, device=x.device, dtype=torch.float32)
    else:
        _check_tensor(out, (n,) + geom.output_shape, "output tensor")
    if n == 0:
        return out
    mode_id = _native.mode_id(mode)
    g = _native.Geom.of(geom, n)
    lib = _native.lib()
    with torch.cuda.device(x.device):
        need = int(lib.smmc_workspace_bytes(ctypes.byref(g), mode_id))
        ws_ptr, ws_len = None, 0
        if need:
            if workspace is None or workspace.numel() * workspace.element_size() < need:
                workspace = torch.zeros(need, dtype=torch.uint8, device=x.device)
            ws_ptr, ws_len = workspace.data_ptr(), workspace.numel() * workspace.element_size()
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _native.check(lib.smmc_conv2d_fwd_f32(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(weights_smm.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), ctypes.byref(g), mode_id,
            ctypes.c_void_p(ws_ptr) if ws_ptr else None, ws_len,
            ctypes.c_void_p(stream) if stream else None), "smmc_conv2d_fwd_f32")
    return out


def conv2d_gather(x, w_slice, outs, geom_local, co_base, co_total, *, workspace=None):
    """Fused output-channel-shard conv + all-gather (``smmc_conv2d_fwd_f32_gather``).

    ``x`` (N, c_i, h, w); ``w_slice`` the compact (c_i, k_w, k_h, c_lo) SMM
    weights of channels [co_base, co_base + c_lo) (``geom_local.out_channels``
    = c_lo); ``outs``: up to 8 destinations of the full (N, co_total, h', w')
    output — CUDA tensors, or raw device addresses (ints) such as peer buffers
    mapped with ``_native.ipc_open``.  Every destination receives this
    shard's channels; launched on torch's current stream, no synchronisation.
    """
    torch = _torch()
    if not isinstance(x, torch.Tensor) or x.dim() != 4:
        raise ShapeMismatchError("x must be a 4-D torch.Tensor (N, c_i, h, w)")
    n = x.shape[0]
    _check_tensor(x, (n,) + geom_local.input_shape, "input batch")
    _check_tensor(w_slice, geom_local.weights_smm_shape, "weight slice")
    if not 1 <= len(outs) <= _native.SMMC_MAX_OUT:
        raise ShapeMismatchError(f"1..{_native.SMMC_MAX_OUT} output replicas required")
    full = (n, co_total, geom_local.out_h, geom_local.out_w)
    ptrs = []
    for o in outs:
        if isinstance(o, int):
            ptrs.append(o)
        else:
            _check_tensor(o, full, "output replica")
            ptrs.append(o.data_ptr())
    if n == 0:
        return
    g = _native.Geom.of(geom_local, n)
    lib = _native.lib()
    with torch.cuda.device(x.device):
        need = int(lib.smmc_gather_workspace_bytes(ctypes.byref(g)))
        ws_ptr, ws_len = None, 0
        if need:
            if workspace is None or workspace.numel() * workspace.element_size() < need:
                workspace = torch.zeros(need, dtype=torch.uint8, device=x.device)
            ws_ptr, ws_len = workspace.data_ptr(), workspace.numel() * workspace.element_size()
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        stream = torch.cuda.current_stream(x.device).cuda_stream
        _native.check(lib.smmc_conv2d_fwd_f32_gather(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w_slice.data_ptr()), arr, len(ptrs),
            ctypes.byref(g), int(co_base), int(co_total),
            ctypes.c_void_p(ws_ptr) if ws_ptr else None, ws_len,
            ctypes.c_void_p(stream) if stream else None), "smmc_conv2d_fwd_f32_gather")


class SmmConv2d:
    """A fitted layer held on one device: weights in SMM order, a reusable
    workspace, and a call that launches on the current stream.

    ``weights`` may be OIHW numpy / torch (repacked once here, untimed).
    """

    def __init__(self, geom, weights, device="cuda", mode="ffma", max_batch=None, autotune=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise DeviceError("SmmConv2d needs a CUDA device (no CPU fallback)")
        self.geom = geom
        self.mode = mode
        self.device = torch.device(device)
        # per-shape autotuning (needs the batch size: plans depend on it); off
        # unless asked for here or by SMMC_AUTOTUNE=1
        self.autotune_report = None
        if autotune is None:
            autotune = _native.autotune_enabled()
        if autotune and max_batch and mode == "ffma":
            with torch.cuda.device(self.device):
                self.autotune_report = _native.autotune(geom, max_batch)
        w = torch.as_tensor(weights, dtype=torch.float32)
        if tuple(w.shape) == geom.weights_shape:
            w = w.permute(1, 3, 2, 0)
        elif tuple(w.shape) != geom.weights_smm_shape:
            raise ShapeMismatchError(
                f"weights must be OIHW {geom.weights_shape} or SMM {geom.weights_smm_shape}")
        self.weights_smm = w.contiguous().to(self.device)
        self._ws = None
        if max_batch:
            self.workspace_for(max_batch)

    def workspace_for(self, batch):
        torch = _torch()
        need = _native.workspace_bytes(self.geom, batch, self.mode)
        if need and (self._ws is None or self._ws.numel() < need):
            self._ws = torch.zeros(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def launches(self, batch):
        return _native.plan_launches(self.geom, batch, self.mode)

    def __call__(self, x, out=None):
        return conv2d(x, self.weights_smm, self.geom, mode=self.mode, out=out,
                      workspace=self.workspace_for(x.shape[0]))


# --------------------------------------------------------------------------
# Separately labelled tensor-core variant: bf16 inputs, fp32 accumulation in
# TMEM (tcgen05), fp32 NCHW output.  Parity bar 2e-2 * max|ref| (BASELINE
# config 5).  Input is channels-last bf16, weights are packed per tap.
# --------------------------------------------------------------------------

def tc_supported(geom, batch=1):
    g = _native.Geom.of(geom, max(batch, 1))
    return bool(_native.lib().smmc_tc_supported(ctypes.byref(g)))


def _stream_ptr(torch, dev):
    s = torch.cuda.current_stream(dev).cuda_stream
    return ctypes.c_void_p(s) if s else None


def packed_input_shape(geom, n):
    """Zero-padded channels-last bf16 layout of the tensor-core variant."""
    return (n, geom.padded_h, geom.padded_w, geom.in_channels)


def pack_input_bf16(x, geom, out=None):
    """fp32 NCHW (N, c_i, h, w) -> zero-padded bf16 NHWC (N, h+2p_h, w+2p_w, c_i)."""
    torch = _torch()
    n = x.shape[0]
    _check_tensor(x, (n,) + geom.input_shape, "input batch")
    if out is None:
        out = torch.empty(packed_input_shape(geom, n), dtype=torch.bfloat16, device=x.device)
    g = _native.Geom.of(geom, n)
    with torch.cuda.device(x.device):
        _native.check(_native.lib().smmc_pack_input_bf16_nhwc(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.byref(g),
            _stream_ptr(torch, x.device)), "smmc_pack_input_bf16_nhwc")
    return out


def pack_weights_bf16(weights_smm, geom):
    """fp32 (c_i, k_w, k_h, c_o) -> bf16 (k_w*k_h, c_o, c_i) on the device."""
    torch = _torch()
    _check_tensor(weights_smm, geom.weights_smm_shape, "repacked weight tensor")
    out = torch.empty((geom.k_w * geom.k_h, geom.out_channels, geom.in_channels),
                      dtype=torch.bfloat16, device=weights_smm.device)
    g = _native.Geom.of(geom, 1)
    with torch.cuda.device(weights_smm.device):
        _native.check(_native.lib().smmc_pack_weights_bf16(
            ctypes.c_void_p(weights_smm.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.byref(g), _stream_ptr(torch, weights_smm.device)), "smmc_pack_weights_bf16")
    return out


def tc_workspace_bytes(geom, batch, split3=False):
    """Scratch of the tensor-core split-K (few-tile layers), else 0."""
    g = _native.Geom.of(geom, batch)
    return int(_native.lib().smmc_tc_workspace_bytes(ctypes.byref(g), 1 if split3 else 0))


def _tc_workspace(torch, geom, n, dev, split3, workspace):
    need = tc_workspace_bytes(geom, n, split3) if n else 0
    if not need:
        return None, 0
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    return ctypes.c_void_p(workspace.data_ptr()), workspace.numel() * workspace.element_size()


def conv2d_bf16_tc(x_nhwc, w_tc, geom, out=None, workspace=None):
    """tcgen05 bf16 conv: x_nhwc zero-padded bf16 (N, h+2p_h, w+2p_w, c_i) from
    pack_input_bf16, w_tc bf16 (taps, c_o, c_i) -> fp32 NCHW (N, c_o, h', w'),
    on torch's current stream.  Few-tile layers split K across CTAs into a
    workspace (passed, or taken from torch's caching allocator)."""
    torch = _torch()
    if not isinstance(x_nhwc, torch.Tensor) or x_nhwc.dim() != 4 or not x_nhwc.is_cuda \
            or x_nhwc.dtype != torch.bfloat16 or not x_nhwc.is_contiguous():
        raise ShapeMismatchError("x_nhwc must be a contiguous CUDA bf16 (N, hp, wp, c_i) tensor")
    n = x_nhwc.shape[0]
    if tuple(x_nhwc.shape) != packed_input_shape(geom, n):
        raise ShapeMismatchError(f"x_nhwc has shape {tuple(x_nhwc.shape)}, expected "
                                 f"{packed_input_shape(geom, n)}")
    if tuple(w_tc.shape) != (geom.k_w * geom.k_h, geom.out_channels, geom.in_channels) \
            or w_tc.dtype != torch.bfloat16 or not w_tc.is_cuda:
        raise ShapeMismatchError("w_tc must be bf16 (k_w*k_h, c_o, c_i) on the device")
    if out is None:
        out = torch.empty((n,) + geom.output_shape, device=x_nhwc.device, dtype=torch.float32)
    else:
        _check_tensor(out, (n,) + geom.output_shape, "output tensor")
    if n == 0:
        return out
    g = _native.Geom.of(geom, n)
    with torch.cuda.device(x_nhwc.device):
        ws, ws_len = _tc_workspace(torch, geom, n, x_nhwc.device, False, workspace)
        _native.check(_native.lib().smmc_conv2d_fwd_bf16_tc_ws(
            ctypes.c_void_p(x_nhwc.data_ptr()), ctypes.c_void_p(w_tc.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), ctypes.byref(g), ws, ws_len,
            _stream_ptr(torch, x_nhwc.device)), "smmc_conv2d_fwd_bf16_tc_ws")
    return out


class TcSmmConv2d:
    """Fitted bf16 tensor-core layer: weights packed once (untimed, like the
    reference's repack); ``pack_input`` casts an fp32 NCHW batch to bf16 NHWC;
    the call runs the tcgen05 kernel."""

    def __init__(self, geom, weights, device="cuda"):
        torch = _torch()
        if not torch.cuda.is_available():
            raise DeviceError("TcSmmConv2d needs a CUDA device (no CPU fallback)")
        if not tc_supported(geom):
            from .errors import BackendUnsupportedError
            raise BackendUnsupportedError(
                "bf16 tensor-core variant needs stride 1 and c_i % 8 == 0")
        self.geom = geom
        self.device = torch.device(device)
        w = torch.as_tensor(weights, dtype=torch.float32)
        if tuple(w.shape) == geom.weights_shape:
            w = w.permute(1, 3, 2, 0)
        w = w.contiguous().to(self.device)
        self.w_tc = pack_weights_bf16(w, geom)
        self._ws = {}

    def pack_input(self, x, out=None):
        return pack_input_bf16(x, self.geom, out=out)

    def __call__(self, x_nhwc, out=None):
        n = x_nhwc.shape[0]
        if n not in self._ws:
            need = tc_workspace_bytes(self.geom, n) if n else 0
            self._ws[n] = (_torch().empty(need, dtype=_torch().uint8, device=self.device)
                           if need else None)
        return conv2d_bf16_tc(x_nhwc, self.w_tc, self.geom, out=out, workspace=self._ws[n])


# --------------------------------------------------------------------------
# fp32-accurate tensor-core path ("bf16x3"): each fp32 operand split into
# bf16 hi + lo; the three significant cross products accumulate in fp32 TMEM
# as one bf16 tcgen05 conv over 3*c_i channels.  fp32 in, fp32 out; parity
# bar the fp32 one (1e-4 * max|ref|).
# --------------------------------------------------------------------------

def packed_input3_shape(geom, n):
    return (n, geom.padded_h, geom.padded_w, 3 * geom.in_channels)


def pack_input_bf16x3(x, geom, out=None):
    """fp32 NCHW -> zero-padded bf16 NHWC with 3*c_i channels [hi | lo | hi]."""
    torch = _torch()
    n = x.shape[0]
    _check_tensor(x, (n,) + geom.input_shape, "input batch")
    if out is None:
        out = torch.empty(packed_input3_shape(geom, n), dtype=torch.bfloat16, device=x.device)
    elif tuple(out.shape) != packed_input3_shape(geom, n) or out.dtype != torch.bfloat16:
        raise ShapeMismatchError("out must be bf16 " + str(packed_input3_shape(geom, n)))
    g = _native.Geom.of(geom, n)
    with torch.cuda.device(x.device):
        _native.check(_native.lib().smmc_pack_input_bf16x3_nhwc(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(out.data_ptr()), ctypes.byref(g),
            _stream_ptr(torch, x.device)), "smmc_pack_input_bf16x3_nhwc")
    return out


def pack_weights_bf16x3(weights_smm, geom):
    """fp32 (c_i, k_w, k_h, c_o) -> bf16 (k_w*k_h, c_o, 3*c_i) [hi | hi | lo]."""
    torch = _torch()
    _check_tensor(weights_smm, geom.weights_smm_shape, "repacked weight tensor")
    out = torch.empty((geom.k_w * geom.k_h, geom.out_channels, 3 * geom.in_channels),
                      dtype=torch.bfloat16, device=weights_smm.device)
    g = _native.Geom.of(geom, 1)
    with torch.cuda.device(weights_smm.device):
        _native.check(_native.lib().smmc_pack_weights_bf16x3(
            ctypes.c_void_p(weights_smm.data_ptr()), ctypes.c_void_p(out.data_ptr()),
            ctypes.byref(g), _stream_ptr(torch, weights_smm.device)), "smmc_pack_weights_bf16x3")
    return out


def conv2d_bf16x3_tc(x3, w3, geom, out=None, workspace=None):
    """tcgen05 split-bf16 conv of pack_input_bf16x3 / pack_weights_bf16x3
    operands -> fp32 NCHW, on torch's current stream."""
    torch = _torch()
    if not isinstance(x3, torch.Tensor) or not x3.is_cuda or x3.dtype != torch.bfloat16 \
            or x3.dim() != 4 or not x3.is_contiguous():
        raise ShapeMismatchError("x3 must be a contiguous CUDA bf16 (N, hp, wp, 3*c_i) tensor")
    n = x3.shape[0]
    if tuple(x3.shape) != packed_input3_shape(geom, n):
        raise ShapeMismatchError(f"x3 has shape {tuple(x3.shape)}, expected "
                                 f"{packed_input3_shape(geom, n)}")
    if tuple(w3.shape) != (geom.k_w * geom.k_h, geom.out_channels, 3 * geom.in_channels) \
            or w3.dtype != torch.bfloat16 or not w3.is_cuda:
        raise ShapeMismatchError("w3 must be bf16 (k_w*k_h, c_o, 3*c_i) on the device")
    if out is None:
        out = torch.empty((n,) + geom.output_shape, device=x3.device, dtype=torch.float32)
    else:
        _check_tensor(out, (n,) + geom.output_shape, "output tensor")
    if n == 0:
        return out
    g = _native.Geom.of(geom, n)
    with torch.cuda.device(x3.device):
        ws, ws_len = _tc_workspace(torch, geom, n, x3.device, True, workspace)
        _native.check(_native.lib().smmc_conv2d_fwd_bf16x3_tc(
            ctypes.c_void_p(x3.data_ptr()), ctypes.c_void_p(w3.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), ctypes.byref(g), ws, ws_len,
            _stream_ptr(torch, x3.device)), "smmc_conv2d_fwd_bf16x3_tc")
    return out


def tc3_plan_describe(geom, batch=1):
    """Plan of the split-bf16 path (the bf16 plan over 3*c_i channels)."""
    from .geometry import ConvGeometry
    g3 = ConvGeometry(3 * geom.in_channels, geom.out_channels, geom.in_h, geom.in_w, geom.k_h,
                      geom.k_w, geom.stride_h, geom.stride_w, geom.pad_h, geom.pad_w)
    return _native.tc_plan_describe(g3, batch)


class Tc3SmmConv2d:
    """Fitted fp32-accurate tensor-core layer (fp32 NCHW in, fp32 NCHW out):
    weights split and packed once (untimed, like the reference's repack); each
    call splits/packs the input batch into a cached bf16 buffer and runs the
    tcgen05 kernel (both inside a timed step)."""

    def __init__(self, geom, weights, device="cuda"):
        torch = _torch()
        if not torch.cuda.is_available():
            raise DeviceError("Tc3SmmConv2d needs a CUDA device (no CPU fallback)")
        if not tc_supported(geom):
            from .errors import BackendUnsupportedError
            raise BackendUnsupportedError(
                "split-bf16 tensor-core path needs stride 1 and c_i % 8 == 0")
        self.geom = geom
        self.device = torch.device(device)
        w = torch.as_tensor(weights, dtype=torch.float32)
        if tuple(w.shape) == geom.weights_shape:
            w = w.permute(1, 3, 2, 0)
        w = w.contiguous().to(self.device)
        self.w3 = pack_weights_bf16x3(w, geom)
        self._x3 = None
        self._ws = None

    def __call__(self, x, out=None):
        torch = _torch()
        n = x.shape[0]
        if self._x3 is None or self._x3.shape[0] != n:
            self._x3 = torch.empty(packed_input3_shape(self.geom, n), dtype=torch.bfloat16,
                                   device=self.device)
            need = tc_workspace_bytes(self.geom, n, split3=True) if n else 0
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device) if need else None
        pack_input_bf16x3(x, self.geom, out=self._x3)
        return conv2d_bf16x3_tc(self._x3, self.w3, self.geom, out=out, workspace=self._ws)


def tc_plan_halo(geom):
    """True when the tensor-core variant uses the halo kernel for this geometry
    (one TMA box per 64-channel block shared by all taps)."""
    halo_rows = 128 + (geom.k_h - 1) * geom.padded_w + (geom.k_w - 1)
    return halo_rows <= 256
