"""Multi-GPU sharding of the conv path (one process per GPU, torch.distributed).

Two partitions, both lifted from the reference:

* batch sharding — samples are independent (Conv2D.transform's per-sample
  loop, estimator.py:123-124): rank r convolves samples [N*r/P, N*(r+1)/P);
  weights are replicated; NO collective on the data path.
* output-channel sharding — the reference's Algorithm 2 partition
  (smm.py:273-279: worker n owns channels [n*ceil(c_o/d), ...)) lifted to
  devices: every rank holds the full input and a W_smm[..., lo:hi] slice,
  computes y_r (N, c_o/P, h', w'), then one all-gather (NCCL over NVLink)
  assembles (N, c_o, h', w').  The gathered buffer is rank-major
  (P, N, c_o/P, h'*w'); a single permute-copy restores NCHW.
* fused output-channel sharding (``shard="cout_fused"``, the product path on
  GPUs): no collective payload at all — every rank maps its peers' full
  output buffers over NVLink (CUDA IPC, exchanged once at construction) and
  the conv's placement pass stores this rank's channels into all of them
  (``smmc_conv2d_fwd_f32_gather``); a 1-element NCCL all-reduce before and
  after is the only cross-rank traffic (write-after-read and read-after-write
  fences).

``conv_fn`` is injectable so the sharding logic is testable on CPU with the
gloo backend (tests/test_parallel.py); on GPU it is ``device.conv2d``.
"""

import torch
import torch.distributed as dist

from .errors import ShapeMismatchError
from .geometry import ConvGeometry

__all__ = ["batch_shard", "cout_shard", "cout_geometry", "all_gather_cout",
           "PeerBuffers", "ShardedSmmConv"]


def batch_shard(n, rank, world):
    """[lo, hi) samples of rank ``rank`` (balanced, contiguous)."""
    return n * rank // world, n * (rank + 1) // world


def cout_shard(c_o, rank, world):
    """[lo, hi) output channels of ``rank``: ceil(c_o/P) per rank, as the
    reference's chunk = ceil(c_o/d) (smm.py:273); trailing ranks may be short
    or empty."""
    chunk = -(-c_o // world)
    lo = min(rank * chunk, c_o)
    return lo, min(lo + chunk, c_o)


def cout_geometry(geom, lo, hi):
    return ConvGeometry(geom.in_channels, hi - lo, geom.in_h, geom.in_w, geom.k_h, geom.k_w,
                        geom.stride_h, geom.stride_w, geom.pad_h, geom.pad_w)


def all_gather_cout(y_local, gather_buf, out, c_o, world, group=None):
    """Assemble the full (N, c_o, h', w') output from per-rank channel slices.

    ``y_local``: (N, c_loc, h', w') with c_loc = ceil(c_o/P) (the last ranks'
    tails are padding and ignored).  ``gather_buf``: (P, N, c_loc, h', w').
    ``out``: (N, c_o, h', w').
    """
    if world == 1:
        out.copy_(y_local[:, :c_o])
        return out
    chunk = y_local.shape[1]
    if gather_buf.shape[0] != world or tuple(gather_buf.shape[1:]) != tuple(y_local.shape):
        raise ShapeMismatchError("gather buffer must be (P,) + y_local.shape")
    n = y_local.shape[0]
    flat = gather_buf.view((world * n,) + tuple(y_local.shape[1:]))
    dist.all_gather_into_tensor(flat, y_local.contiguous(), group=group)
    full = gather_buf.permute(1, 0, 2, 3, 4).reshape(n, world * chunk, *y_local.shape[2:])
    out.copy_(full[:, :c_o])
    return out


class PeerBuffers:
    """Every rank's copy of one output buffer, as device addresses usable by
    this rank's kernels: its own ``data_ptr()`` plus the peers' buffers opened
    through CUDA IPC (handles exchanged with ``all_gather_object``).  Order:
    rank 0 .. P-1.  ``ipc`` is injectable for CPU tests."""

    def __init__(self, out, group=None, ipc=None):
        from . import _native
        self.ipc = ipc or _native
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.out = out
        mine = self.ipc.ipc_handle(out.data_ptr()) if self.world > 1 else (b"", 0)
        entries = [None] * self.world
        if self.world > 1:
            dist.all_gather_object(entries, mine, group=group)
        else:
            entries[0] = mine
        self.ptrs, self._opened = [], []
        for r, (handle, offset) in enumerate(entries):
            if r == self.rank:
                self.ptrs.append(out.data_ptr())
            else:
                ptr = self.ipc.ipc_open(handle, offset)
                self._opened.append((ptr, offset))
                self.ptrs.append(ptr)

    def close(self):
        for ptr, offset in self._opened:
            self.ipc.ipc_close(ptr, offset)
        self._opened = []


class ShardedSmmConv:
    """One conv layer sharded over the default process group.

    ``shard="batch"``: forward(x_local) -> y_local, no collective.
    ``shard="cout"``:  forward(x_full)  -> y_full via all-gather.
    ``shard="cout_fused"``: forward(x_full) -> y_full written by every rank's
    conv straight into every rank's output over NVLink (``batch`` fixes the
    output buffer, or pass ``out``; ``gather_fn`` / ``ipc`` are injectable for
    CPU tests).
    ``weights_smm`` is the full (c_i, k_w, k_h, c_o) tensor on this rank's device.
    """

    def __init__(self, geom, weights_smm, shard="batch", conv_fn=None, mode="ffma",
                 batch=None, gather_fn=None, ipc=None, out=None):
        if shard not in ("batch", "cout", "cout_fused"):
            raise ValueError("shard must be 'batch', 'cout' or 'cout_fused'")
        self.geom = geom
        self.shard = shard
        self.mode = mode
        self.world = dist.get_world_size() if dist.is_initialized() else 1
        self.rank = dist.get_rank() if dist.is_initialized() else 0
        if conv_fn is None:
            from .device import conv2d

            def conv_fn(x, w, g):
                return conv2d(x, w, g, mode=mode)
        self.conv_fn = conv_fn
        if tuple(weights_smm.shape) != geom.weights_smm_shape:
            raise ShapeMismatchError("weights must be in SMM order (c_i, k_w, k_h, c_o)")
        if shard == "cout_fused":
            if mode != "ffma":
                raise ValueError("cout_fused runs the ffma mode")
            if not batch or batch < 1:
                raise ValueError("cout_fused needs the batch size of its output buffer")
            if gather_fn is None:
                from .device import conv2d_gather as gather_fn
            self.gather_fn = gather_fn
            self.lo, self.hi = cout_shard(geom.out_channels, self.rank, self.world)
            self.local_geom = (cout_geometry(geom, self.lo, self.hi)
                               if self.hi > self.lo else None)
            self.weights = weights_smm[..., self.lo:self.hi].contiguous()
            shape = (batch,) + geom.output_shape
            if out is None:
                out = torch.empty(shape, dtype=weights_smm.dtype, device=weights_smm.device)
            elif tuple(out.shape) != shape or not out.is_contiguous():
                raise ShapeMismatchError(f"out must be a contiguous {shape} tensor")
            self.out = out
            self.peers = PeerBuffers(self.out, ipc=ipc)
            self._flag = torch.zeros(1, dtype=torch.float32, device=weights_smm.device)
            self._flag_host = torch.zeros(1, dtype=torch.float32)
            return
        if shard == "cout":
            self.chunk = -(-geom.out_channels // self.world)
            lo, hi = cout_shard(geom.out_channels, self.rank, self.world)
            w = weights_smm[..., lo:hi]
            if hi - lo < self.chunk:  # pad the short tail rank with zero channels
                pad = torch.zeros(w.shape[:-1] + (self.chunk - (hi - lo),),
                                  dtype=w.dtype, device=w.device)
                w = torch.cat([w, pad], dim=-1)
            self.local_geom = cout_geometry(geom, 0, self.chunk)
            self.weights = w.contiguous()
        else:
            self.local_geom = geom
            self.weights = weights_smm.contiguous()

    def _fence(self):
        """Cross-rank ordering point of the fused gather.  NCCL: a 1-element
        all-reduce on the compute stream (stream-ordered, no host sync).
        Other backends (gloo -- e.g. several ranks sharing one GPU, which
        NCCL refuses): drain this rank's device work, then all-reduce a host
        flag, so no rank passes the fence before every rank's writes landed."""
        if self.world <= 1:
            return
        if self._flag.is_cuda and dist.get_backend() != "nccl":
            torch.cuda.synchronize(self._flag.device)
            dist.all_reduce(self._flag_host)
        else:
            dist.all_reduce(self._flag)

    def forward(self, x):
        if self.shard == "cout_fused":
            if x.shape[0] != self.out.shape[0]:
                raise ShapeMismatchError(
                    f"cout_fused was built for batch {self.out.shape[0]}, got {x.shape[0]}")
            self._fence()  # peers are done reading the previous output
            if self.local_geom is not None:
                self.gather_fn(x, self.weights, self.peers.ptrs, self.local_geom, self.lo,
                               self.geom.out_channels)
            self._fence()  # every shard has landed in every replica
            return self.out
        y_local = self.conv_fn(x, self.weights, self.local_geom)
        if self.shard == "batch":
            return y_local
        n = x.shape[0]
        buf = torch.empty((self.world,) + tuple(y_local.shape), dtype=y_local.dtype,
                          device=y_local.device)
        out = torch.empty((n,) + self.geom.output_shape, dtype=y_local.dtype,
                          device=y_local.device)
        return all_gather_cout(y_local, buf, out, self.geom.out_channels, self.world)

    __call__ = forward
