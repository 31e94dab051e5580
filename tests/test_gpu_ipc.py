"""The fused c_o-shard gather across REAL processes.

Two (or three) processes share the one GPU this build can lease: each is a
rank of a gloo process group (NCCL refuses two ranks on one device), maps its
peers' output buffers through CUDA IPC (``smmc_ipc_handle`` /
``smmc_ipc_open`` -- a different process may open a handle of the same
device) and runs ``ShardedSmmConv(shard="cout_fused")``: its conv's placement
pass stores its channel slice into every rank's output.  No rank's kernel
waits on another's (the fences are host-side), so this is safe on one GPU.
Every replica must equal the oracle (fp32 tolerance), the replicas must be
bitwise identical, and they must equal the single-process emulation of the
same ranks bitwise (same kernel, same plan).  A second forward over a new
input checks the write-after-read fence."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, geom_t, n, seeds, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    from paper_2411_15659_b200 import ConvGeometry
    from paper_2411_15659_b200.parallel import ShardedSmmConv
    from paper_2411_15659_b200.tensors import synthetic_layer
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = ConvGeometry(*geom_t)
        outs = []
        conv = None
        for seed in seeds:
            x, w = synthetic_layer(g, n, seed)
            ws = torch.from_numpy(np.ascontiguousarray(w.transpose(1, 3, 2, 0))).cuda()
            if conv is None:
                conv = ShardedSmmConv(g, ws, shard="cout_fused", batch=n)
            else:  # same layer, new weights slice (same shard)
                conv.weights = ws[..., conv.lo:conv.hi].contiguous()
            y = conv(torch.from_numpy(x).cuda())
            torch.cuda.synchronize()
            outs.append(y.cpu().numpy().copy())
        q.put((rank, outs, conv.peers.ptrs != [conv.out.data_ptr()]))
        dist.barrier()
        conv.peers.close()
    finally:
        dist.destroy_process_group()


def _run(world, geom_t, n, seeds):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, geom_t, n, seeds, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, outs, mapped = q.get(timeout=240)
            res[r] = (outs, mapped)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.exitcode is None:
                p.kill()
    assert all(p.exitcode == 0 for p in procs)
    return res


def _emulated(g, n, seed, world):
    import torch

    from paper_2411_15659_b200 import device
    from paper_2411_15659_b200.parallel import cout_geometry, cout_shard
    from paper_2411_15659_b200.tensors import synthetic_layer
    x, w = synthetic_layer(g, n, seed)
    ws = np.ascontiguousarray(w.transpose(1, 3, 2, 0))
    xd = torch.from_numpy(x).cuda()
    out = torch.full((n,) + g.output_shape, float("nan"), device="cuda")
    for r in range(world):
        lo, hi = cout_shard(g.out_channels, r, world)
        if hi > lo:
            wd = torch.from_numpy(np.ascontiguousarray(ws[..., lo:hi])).cuda()
            device.conv2d_gather(xd, wd, [out], cout_geometry(g, lo, hi), lo, g.out_channels)
    torch.cuda.synchronize()
    return x, w, out.cpu().numpy()


CASES = [
    ("cfg5_512@7_n8", (512, 512, 7, 7, 3, 3, 1, 1, 1, 1), 8, 2),
    ("odd_c37_p3", (24, 37, 11, 9, 3, 3, 1, 1, 1, 1), 3, 3),
]


@pytest.mark.parametrize("name,geom_t,n,world", CASES, ids=[c[0] for c in CASES])
def test_cout_fused_across_processes(name, geom_t, n, world):
    from oracle import smm_oracle as orc
    from paper_2411_15659_b200 import ConvGeometry
    g = ConvGeometry(*geom_t)
    seeds = [5003, 77]
    res = _run(world, geom_t, n, seeds)
    assert all(mapped for _, mapped in res.values()), "peer buffers were not IPC-mapped"
    for si, seed in enumerate(seeds):
        x, w, emu = _emulated(g, n, seed, world)
        ref = orc.smm_conv_c(x, orc.repack(w), g, threads=orc.host_threads())
        reps = [res[r][0][si] for r in range(world)]
        for y in reps:
            assert np.isfinite(y).all()
            assert orc.max_abs_ratio(y, ref) <= TOL
            assert np.array_equal(y, reps[0])
        assert np.array_equal(reps[0], emu)
