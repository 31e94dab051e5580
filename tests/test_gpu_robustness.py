"""GPU robustness of the C ABI: re-entrancy, stream ordering, graph capture,
workspace contracts, large index ranges and error paths."""

import ctypes
import threading

import numpy as np
import pytest

from oracle import smm_oracle as orc
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, _native
from paper_2411_15659_b200.tensors import synthetic_layer

pytestmark = pytest.mark.gpu
TOL = 1e-4


def test_host_entry_is_reentrant_across_threads():
    """Eight Python threads hammer the host-buffer entry with different
    geometries; every result must still match the oracle (the per-device
    staging pool is mutex-protected, the ctypes call releases the GIL)."""
    geoms = [ConvGeometry(8 + 8 * (i % 3), 16, 10 + i, 12, 3, 3, pad_h=1, pad_w=1) for i in range(8)]
    data = [synthetic_layer(g, 2, 50 + i) for i, g in enumerate(geoms)]
    refs = [orc.smm_conv_c(x, orc.repack(w), g) for g, (x, w) in zip(geoms, data)]
    errors = []

    def work(i):
        g = geoms[i]
        x, w = data[i]
        ws = smm.repack_weights(w, g)
        for _ in range(5):
            y = smm.smm_conv_batched(x, ws, g)
            if orc.max_abs_ratio(y, refs[i]) > TOL:
                errors.append(i)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors


def test_device_path_on_side_stream_and_in_cuda_graph():
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(64, 64, 14, 14, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 4, 9)
    ref = orc.smm_conv_c(x, orc.repack(w), g)
    mod = device.SmmConv2d(g, w, max_batch=4)
    xd = torch.from_numpy(x).cuda()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        y = mod(xd)
    torch.cuda.current_stream().wait_stream(s)
    assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL
    # capture (split-K plans included: the counter memset is a graph node)
    out = torch.empty_like(y)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        mod(xd, out=out)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, y)


def test_workspace_contract_errors():
    import torch
    g = ConvGeometry(512, 512, 7, 7, 3, 3, pad_h=1, pad_w=1)
    need = _native.workspace_bytes(g, 1)
    assert need > 0
    x = torch.zeros((1,) + g.input_shape, device="cuda")
    w = torch.zeros(g.weights_smm_shape, device="cuda")
    y = torch.empty((1,) + g.output_shape, device="cuda")
    lib = _native.lib()
    G = _native.Geom.of(g, 1)
    small = torch.empty(need // 2, dtype=torch.uint8, device="cuda")
    st = lib.smmc_conv2d_fwd_f32(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                 ctypes.c_void_p(y.data_ptr()), ctypes.byref(G), 0,
                                 ctypes.c_void_p(small.data_ptr()), small.numel(), None)
    assert st == _native.SMMC_EWORKSPACE
    with pytest.raises(ValueError):
        _native.check(st)
    # misaligned pointers are rejected before any launch (x needs 4 bytes,
    # w 16 bytes, y 16 bytes when h'*w' % 4 == 0 — here 49: 4 bytes)
    for dx, dw, dy in ((2, 0, 0), (0, 4, 0), (0, 0, 2)):
        st = lib.smmc_conv2d_fwd_f32(ctypes.c_void_p(x.data_ptr() + dx),
                                     ctypes.c_void_p(w.data_ptr() + dw),
                                     ctypes.c_void_p(y.data_ptr() + dy), ctypes.byref(G), 0, None, 0,
                                     None)
        assert st == _native.SMMC_ESHAPE
    st = lib.smmc_conv2d_fwd_f32(None, None, None, ctypes.byref(G), 0, None, 0, None)
    assert st == _native.SMMC_ESHAPE
    st = lib.smmc_conv2d_fwd_f32(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
                                 ctypes.c_void_p(y.data_ptr()), ctypes.byref(G), 7, None, 0, None)
    assert st == _native.SMMC_EUNSUPPORTED


def test_large_index_ranges():
    """A batch whose tensors exceed 2^31 bytes (x: 2.2 GB): 64-bit offsets in
    the loaders and epilogue; checked on first/last samples."""
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(64, 64, 112, 112, 3, 3, pad_h=1, pad_w=1)
    n = 700  # 700*64*112*112*4 B = 2.25 GB per tensor
    assert n * g.in_channels * g.in_h * g.in_w * 4 > 2 ** 31
    torch.manual_seed(0)
    xd = torch.rand((n,) + g.input_shape, device="cuda") * 2 - 1
    _, w = synthetic_layer(ConvGeometry(64, 64, 4, 4, 3, 3, pad_h=1, pad_w=1), 1, 3)
    wd = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    y = device.conv2d(xd, wd, g)
    torch.cuda.synchronize()
    for s in (0, n - 1):
        ref = orc.smm_conv_c(xd[s].cpu().numpy(), orc.repack(w), g, threads=orc.host_threads())
        assert orc.max_abs_ratio(y[s].cpu().numpy(), ref) <= TOL
    del xd, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("gt", [
    (3, 4, 33, 31, 3, 3, 3, 3, 2, 1),      # stride 3, rectangular, c_o % 4 == 0
    (16, 6, 20, 20, 5, 3, 2, 1, 0, 2),     # c_o % 4 != 0 on the tap-major path
    (17, 9, 15, 13, 4, 2, 1, 2, 3, 0),     # even kernel, c_i % 16 != 0, stride (1,2)
    (32, 40, 9, 9, 9, 9, 1, 1, 4, 4),      # 9x9 kernel (generic tap path)
    (2, 3, 40, 5, 35, 1, 1, 1, 0, 0),      # k_h = 35 > 32: no padding masks (division path)
])
def test_unusual_geometries(gt):
    import torch
    from paper_2411_15659_b200 import device
    g = ConvGeometry(*gt)
    x, w = synthetic_layer(g, 3, 21)
    ws = smm.repack_weights(w, g)
    ref = orc.smm_conv_c(x, orc.repack(w), g)
    y = device.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(ws).cuda(), g)
    assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL
    ye = smm.smm_conv_batched(x, ws, g, mode="exact")
    assert np.array_equal(ye, ref)


def test_pinned_host_buffers():
    """smmc_host_alloc_pinned: page-locked, usable by the host entry, freed
    with the array; foreign pointers are rejected."""
    import gc
    import torch
    g = ConvGeometry(16, 24, 12, 10, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 3, 8)
    xp = _native.pinned_copy(x)
    wp = _native.pinned_copy(smm.repack_weights(w, g))
    assert torch.from_numpy(xp).is_pinned() and xp.ctypes.data % (2 << 20) == 0
    y = smm.smm_conv_batched(xp, wp, g)
    assert orc.max_abs_ratio(y, orc.smm_conv_c(x, orc.repack(w), g)) <= TOL
    del xp, wp
    gc.collect()
    assert _native.lib().smmc_host_free_pinned(ctypes.c_void_p(12345 * 4096)) == _native.SMMC_ESHAPE


@pytest.mark.parametrize("gt,n", [
    ((256, 200, 7, 7, 3, 3, 1, 1, 1, 1), 2),    # 2 channel chunks (128 + 72)
    ((512, 512, 7, 7, 3, 3, 1, 1, 1, 1), 1),    # config 2 N=1: 8 chunks of 64
    ((128, 96, 5, 6, 5, 3, 1, 2, 2, 1), 3),     # rectangular kernel, stride (1, 2)
    ((64, 70, 4, 4, 1, 1, 1, 1, 0, 0), 1),      # c_o % 32 != 0, 1x1
    ((40, 256, 3, 3, 3, 3, 1, 1, 1, 1), 1),     # c_i % 16 != 0: batch pipeline instead
    ((96, 64, 6, 6, 3, 3, 1, 1, 1, 1), 2),      # 96 channels -> chunks of 48
])
def test_host_entry_weight_heavy_layers(gt, n):
    """Weight-dominated layers through the host entry (weights uploaded in one
    copy ahead of the batch chunks; chunked weight uploads measured slower)."""
    g = ConvGeometry(*gt)
    x, w = synthetic_layer(g, n, 31)
    ws = smm.repack_weights(w, g)
    assert ws.size > x.size + n * g.out_channels * g.out_h * g.out_w  # really weight-heavy
    y = smm.smm_conv_batched(_native.pinned_copy(x), _native.pinned_copy(ws), g)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    assert orc.max_abs_ratio(y, ref) <= TOL
    # exact mode on the same shape keeps the batch pipeline and stays bitwise
    ye = smm.smm_conv_batched(x, ws, g, mode="exact")
    assert np.array_equal(ye, ref)


def test_host_entry_multi_chunk_odd_sample_sizes():
    """Batch chunks of a sample size that is not a multiple of 4 floats
    (11x11 s4 stem: 3*227*227 inputs, 55*55 outputs per plane): chunk
    pointers are only 4-byte aligned, the kernel's scalar paths take them."""
    g = ConvGeometry(3, 96, 227, 227, 11, 11, stride_h=4, stride_w=4)
    n = 8
    x, w = synthetic_layer(g, n, 77)
    ws = smm.repack_weights(w, g)
    y = smm.smm_conv_batched(_native.pinned_copy(x), _native.pinned_copy(ws), g)
    for s in (0, 3, n - 1):
        ref = orc.smm_conv_c(np.ascontiguousarray(x[s:s + 1]), orc.repack(w), g,
                             threads=orc.host_threads())
        assert orc.max_abs_ratio(y[s:s + 1], ref) <= TOL


def test_device_path_unaligned_input_window():
    """x may start at any 4-byte boundary (e.g. a sample slice of an odd-sized
    batch); y keeps 16 bytes when its planes are float4-stored."""
    import torch
    g = ConvGeometry(3, 16, 9, 9, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 3, 4)
    ws = torch.from_numpy(smm.repack_weights(w, g)).cuda()
    xd = torch.from_numpy(x).cuda().reshape(-1)
    lib = _native.lib()
    G = _native.Geom.of(g, 2)
    y = torch.empty((2,) + g.output_shape, device="cuda")
    per = g.in_channels * g.in_h * g.in_w  # 243 floats: odd
    _native.check(lib.smmc_conv2d_fwd_f32(ctypes.c_void_p(xd.data_ptr() + 4 * per),
                                          ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(y.data_ptr()),
                                          ctypes.byref(G), 0, None, 0, None), "conv")
    torch.cuda.synchronize()
    ref = orc.smm_conv_c(np.ascontiguousarray(x[1:]), orc.repack(w), g)
    assert orc.max_abs_ratio(y.cpu().numpy(), ref) <= TOL


def test_fitted_layer_api():
    """smmc_layer: weights uploaded once; forward on host buffers equals the
    per-call host entry bitwise (same plans), for several batch sizes and
    both modes; the estimator's transform goes through it."""
    from paper_2411_15659_b200 import Conv2D
    g = ConvGeometry(32, 48, 14, 14, 3, 3, pad_h=1, pad_w=1)
    x, w = synthetic_layer(g, 9, 12)
    ws = smm.repack_weights(w, g)
    layer = _native.Layer(ws, g)
    for n in (1, 4, 9, 0):
        xs = np.ascontiguousarray(x[:n])
        y = np.full((n,) + g.output_shape, np.nan, np.float32)
        layer.forward(xs, y)
        if n:
            assert np.array_equal(y, smm.smm_conv_batched(xs, ws, g))
    ye = np.empty((3,) + g.output_shape, np.float32)
    layer.forward(np.ascontiguousarray(x[:3]), ye, mode="exact")
    assert np.array_equal(ye, orc.smm_conv_c(np.ascontiguousarray(x[:3]), orc.repack(w), g))
    layer.close()
    layer.close()  # idempotent
    est = Conv2D(out_channels=48, kernel_size=3, padding=1, weights=w).fit(x)
    a = est.transform(x)
    assert np.array_equal(a, est.transform(x))  # cached device weights
    assert orc.max_abs_ratio(a, orc.smm_conv_c(x, orc.repack(w), g)) <= TOL
    est.set_params(weights=np.zeros_like(w)).fit(x)  # refit replaces the device copy
    assert float(np.abs(est.transform(x)).max()) == 0.0
    import pickle
    assert pickle.loads(pickle.dumps(est)).transform(x).shape == a.shape


def test_fitted_layer_async_forward():
    """smmc_layer_forward_host_async: several layers in flight at once on
    their own staging buffers/streams (pinned and pageable host buffers),
    a second call on a busy layer, and close() with work pending -- results
    equal the synchronous entry bitwise."""
    layers = []
    for gt, n, seed in (((64, 64, 28, 28, 3, 3, 1, 1, 1, 1), 6, 1),
                        ((128, 256, 14, 14, 3, 3, 1, 1, 1, 1), 3, 2),
                        ((3, 64, 64, 64, 3, 3, 1, 1, 1, 1), 4, 3),
                        ((32, 16, 9, 9, 1, 1, 1, 1, 0, 0), 2, 4)):
        g = ConvGeometry(*gt)
        x, w = synthetic_layer(g, n, seed)
        ws = smm.repack_weights(w, g)
        L = _native.Layer(ws, g)
        ref = np.empty((n,) + g.output_shape, np.float32)
        L.forward(x, ref)
        layers.append((L, _native.pinned_copy(x), x, ref,
                       _native.pinned_empty((n,) + g.output_shape), np.empty_like(ref)))
    for L, xp, x, _, yp, y in layers:
        L.forward_async(xp, yp)
    for L, xp, x, _, yp, y in layers:      # second call on each busy layer (pageable buffers)
        L.forward_async(x, y)
    for L, *_ in layers:
        L.wait()
        L.wait()                           # idempotent
    for L, xp, x, ref, yp, y in layers:
        assert np.array_equal(yp, ref) and np.array_equal(y, ref)
    layers[0][0].forward_async(layers[0][1], layers[0][4])
    for L, *_ in layers:                   # destroy with work in flight: waits first
        L.close()
    assert np.array_equal(layers[0][4], layers[0][3])


_FIRST_CALL = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2411_15659_b200 as smm
from paper_2411_15659_b200 import ConvGeometry, _native
d = np.load(sys.argv[2])
g = ConvGeometry(*[int(v) for v in d["geom"]])
xp, wp = _native.pinned_copy(d["x"]), _native.pinned_copy(d["ws"])
if sys.argv[3] == "busy":  # ~40 ms of unrelated work queued on the legacy default stream
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    a = torch.randn(4096, 4096, device="cuda")
    for _ in range(20):
        a = a @ a * 1e-3
y = smm.smm_conv_batched(xp, wp, g)
err = float(np.abs(y.astype(np.float64) - d["ref"]).max() / np.abs(d["ref"]).max())
print("ERR", err)
"""


@pytest.mark.parametrize("gt,n", [((512, 512, 7, 7, 3, 3, 1, 1, 1, 1), 1),
                                  ((256, 256, 14, 14, 3, 3, 1, 1, 1, 1), 1)])
def test_host_entry_first_call_in_fresh_process(gt, n, tmp_path):
    """The first host-entry call of a process allocates the staging pool and
    zeroes the split-K workspace; with page-locked inputs the conv starts
    almost at once.  The zeroing must be ordered before the conv on the
    pool's (non-blocking) compute stream -- a legacy-stream cudaMemset was
    not: queued behind other work on the legacy default stream ("busy": a
    torch GEMM chain), it zeroed the conv's partial tiles."""
    import subprocess
    import sys
    from pathlib import Path
    g = ConvGeometry(*gt)
    x, w = synthetic_layer(g, n, 31)
    ws = smm.repack_weights(w, g)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
    f = tmp_path / "case.npz"
    np.savez(f, x=x, ws=ws, ref=ref.astype(np.float64), geom=np.array(gt))
    root = str(Path(__file__).resolve().parents[1])
    for mode in ("idle", "busy", "idle", "busy"):
        out = subprocess.run([sys.executable, "-c", _FIRST_CALL, root, str(f), mode],
                             capture_output=True, text=True, timeout=180)
        assert out.returncode == 0, out.stderr[-2000:]
        err = float(out.stdout.split("ERR")[-1])
        assert err <= TOL, err
