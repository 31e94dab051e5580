"""Multi-process sharding logic on CPU (gloo, world_size 2 and 3).

The local compute is injected (the CPU oracle stands in for the GPU kernel,
which cannot run here); what is under test is the partitioning and the
all-gather/permute that assemble the NCHW output — the host-side logic of the
N>1 path.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_15659_b200 import ConvGeometry
from paper_2411_15659_b200.parallel import (ShardedSmmConv, batch_shard, cout_shard)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_conv(x, w_smm, g):
    from oracle import smm_oracle as orc
    y = orc.smm_conv_c(x.numpy(), w_smm.numpy(), g, threads=1)
    return torch.from_numpy(y)


def _worker(rank, world, port, shard, geom_t, n, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_15659_b200.tensors import synthetic_layer
        g = ConvGeometry(*geom_t)
        x, w = synthetic_layer(g, n, seed=5)
        ws = torch.from_numpy(np.ascontiguousarray(w.transpose(1, 3, 2, 0)))
        conv = ShardedSmmConv(g, ws, shard=shard, conv_fn=_oracle_conv)
        if shard == "batch":
            lo, hi = batch_shard(n, rank, world)
            y = conv(torch.from_numpy(x[lo:hi]))
            parts = [None] * world
            dist.all_gather_object(parts, y.numpy())
            y_full = np.concatenate(parts)
        else:
            y_full = conv(torch.from_numpy(x)).numpy()
        if rank == 0:
            q.put(y_full)
    finally:
        dist.destroy_process_group()


def _run(world, shard, geom_t, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shard, geom_t, n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return y


def _reference(geom_t, n):
    from oracle import smm_oracle as orc
    from paper_2411_15659_b200.tensors import synthetic_layer
    g = ConvGeometry(*geom_t)
    x, w = synthetic_layer(g, n, seed=5)
    return orc.smm_conv_c(x, orc.repack(w), g)


def test_shard_ranges():
    assert [batch_shard(10, r, 4) for r in range(4)] == [(0, 2), (2, 5), (5, 7), (7, 10)]
    assert [cout_shard(512, r, 8) for r in range(8)][-1] == (448, 512)
    assert [cout_shard(10, r, 4) for r in range(4)] == [(0, 3), (3, 6), (6, 9), (9, 10)]
    assert cout_shard(3, 3, 4) == (3, 3)


@pytest.mark.parametrize("world", [2, 3])
def test_batch_sharded_matches_unsharded(world):
    geom_t = (6, 8, 9, 9, 3, 3, 1, 1, 1, 1)
    y = _run(world, "batch", geom_t, n=5)
    assert np.array_equal(y, _reference(geom_t, 5))


@pytest.mark.parametrize("world", [2, 3])
def test_cout_sharded_allgather_matches_unsharded(world):
    # c_o = 10 does not divide by 3: exercises the zero-padded tail rank
    geom_t = (4, 10, 7, 7, 3, 3, 1, 1, 1, 1)
    y = _run(world, "cout", geom_t, n=3)
    assert np.array_equal(y, _reference(geom_t, 3))


# ---- fused c_o-shard gather: the peer-write protocol on CPU.  Shared-memory
# tensors stand in for the NVLink-mapped peer buffers; the injected ipc maps a
# rank's buffer to a handle and back, the injected gather_fn plays the
# smmc_conv2d_fwd_f32_gather placement (oracle conv of this rank's channel
# slice stored into every replica).  The gloo all-reduce fences are real.

class _ShmIpc:
    def __init__(self, bufs):
        self.bufs = bufs

    def ipc_handle(self, ptr):
        idx = [b.data_ptr() for b in self.bufs].index(ptr)
        return bytes([idx]) * 64, 8 * idx

    def ipc_open(self, handle, offset):
        assert offset == 8 * handle[0]
        return self.bufs[handle[0]].data_ptr()

    def ipc_close(self, ptr, offset):
        pass


def _fused_worker(rank, world, port, geom_t, n, bufs, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_15659_b200.tensors import synthetic_layer
        g = ConvGeometry(*geom_t)
        x, w = synthetic_layer(g, n, seed=5)
        ws = torch.from_numpy(np.ascontiguousarray(w.transpose(1, 3, 2, 0)))
        by_ptr = {b.data_ptr(): b for b in bufs}
        calls = []

        def gather_fn(xx, w_slice, ptrs, gl, co_base, co_total):
            calls.append((len(ptrs), co_base, gl.out_channels))
            y = _oracle_conv(xx, w_slice, gl)
            for p in ptrs:
                by_ptr[p][:, co_base:co_base + gl.out_channels] = y

        conv = ShardedSmmConv(g, ws, shard="cout_fused", batch=n, gather_fn=gather_fn,
                              ipc=_ShmIpc(bufs), out=bufs[rank])
        assert conv.peers.ptrs == [b.data_ptr() for b in bufs]
        y = conv(torch.from_numpy(x))
        lo, hi = cout_shard(g.out_channels, rank, world)
        assert calls == ([(world, lo, hi - lo)] if hi > lo else [])
        q.put((rank, y.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,geom_t,n", [
    (2, (6, 8, 9, 7, 3, 3, 1, 1, 1, 1), 2),
    (3, (5, 4, 8, 8, 3, 3, 1, 1, 1, 1), 3),   # c_o = 4 over 3 ranks: rank 2 owns nothing
])
def test_cout_fused_peer_write_protocol(world, geom_t, n):
    from oracle import smm_oracle as orc
    from paper_2411_15659_b200.tensors import synthetic_layer
    g = ConvGeometry(*geom_t)
    bufs = [torch.full((n,) + g.output_shape, float("nan")).share_memory_() for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, geom_t, n, bufs, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get() for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    x, w = synthetic_layer(g, n, seed=5)
    ref = orc.smm_conv_c(x, orc.repack(w), g, threads=1)
    for r in range(world):
        np.testing.assert_array_equal(got[r], ref)      # each rank's returned output
        np.testing.assert_array_equal(bufs[r].numpy(), ref)  # and every replica


def test_cout_fused_argument_errors():
    g = ConvGeometry(4, 8, 6, 6, 3, 3, pad_h=1, pad_w=1)
    ws = torch.zeros(g.weights_smm_shape)
    with pytest.raises(ValueError):
        ShardedSmmConv(g, ws, shard="cout_fused")            # no batch
    with pytest.raises(ValueError):
        ShardedSmmConv(g, ws, shard="cout_fused", batch=2, mode="exact")
    from paper_2411_15659_b200 import ShapeMismatchError
    with pytest.raises(ShapeMismatchError):
        ShardedSmmConv(g, ws, shard="cout_fused", batch=2, gather_fn=lambda *a: None,
                       out=torch.empty(3, 8, 6, 6))
    conv = ShardedSmmConv(g, ws, shard="cout_fused", batch=2, gather_fn=lambda *a: None)
    with pytest.raises(ShapeMismatchError):
        conv(torch.zeros(3, 4, 6, 6))
