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
