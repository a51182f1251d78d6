"""Sharded PCF Learned Sort over R GPUs.

One process per GPU; rank r holds a contiguous shard of the global array.  The
library (``pcf_shard_*`` in include/pcf_sort.h, kernels in csrc/pcf_shard.cuh)
runs every step of the method; this module only issues the collectives between
the calls -- NCCL over NVLink / NVSwitch through ``torch.distributed`` in
production (``TorchComm``):

  1. pcf_shard_minmax      -> all-reduce MIN / MAX of the extremes, MAX of the NaN flag
  2. pcf_shard_counts      -> all-reduce SUM of the level-1 per-bin sample counts
  3. pcf_shard_histogram   -> all-gather of the shards' bucket histograms
  4. pcf_shard_partition   -> all-to-all of the keys, bucket range r to rank r
  5. pcf_shard_sort_range  -> rank r's sorted slice of the global output

The result is Algorithm 1 on the whole array: every rank's
slice is the single-GPU output's slice and every node record is the single-GPU
one (the level-1 record on rank 0).  ``LoopbackComm`` runs R ranks as threads of
one process (each on its own CUDA stream) with host-side exchanges: the test
harness for one GPU, where no rank's kernel ever waits on another's.
"""
from __future__ import annotations

import ctypes
import threading

from . import KEY_F64, KEY_U64, FLAG_SYNC, FLAG_SAMPLE_ALL, NODE_DTYPE, PassLog, _check, lib, make_params

__all__ = ["TorchComm", "LoopbackHub", "LoopbackComm", "sort_sharded", "ShardInfo"]


class ShardC(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint64), ("offset", ctypes.c_uint64), ("R", ctypes.c_uint32),
                ("rank", ctypes.c_uint32), ("state", ctypes.c_void_p), ("state_bytes", ctypes.c_size_t)]


def _bind():
    L = lib()
    if getattr(L, "_shard_bound", False):
        return L
    vp, sz, i32, u32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64
    SP = ctypes.POINTER(ShardC)
    L.pcf_shard_state_bytes.argtypes = [u64, u32]; L.pcf_shard_state_bytes.restype = sz
    L.pcf_shard_workspace_bytes.argtypes = [sz, u64]; L.pcf_shard_workspace_bytes.restype = sz
    L.pcf_shard_views.argtypes = [SP, ctypes.POINTER(vp), ctypes.POINTER(u64)]; L.pcf_shard_views.restype = i32
    L.pcf_shard_minmax.argtypes = [vp, sz, i32, SP, vp]; L.pcf_shard_minmax.restype = i32
    PP = ctypes.c_void_p
    L.pcf_shard_counts.argtypes = [vp, sz, i32, SP, PP, vp]; L.pcf_shard_counts.restype = i32
    L.pcf_shard_histogram.argtypes = [vp, sz, i32, SP, PP, vp]; L.pcf_shard_histogram.restype = i32
    L.pcf_shard_partition.argtypes = [vp, sz, i32, SP, vp, ctypes.POINTER(u64), ctypes.POINTER(u64),
                                      ctypes.POINTER(u64), vp]
    L.pcf_shard_partition.restype = i32
    L.pcf_shard_sort_range.argtypes = [vp, vp, sz, i32, SP, ctypes.POINTER(u64), PP, vp]
    L.pcf_shard_sort_range.restype = i32
    L._shard_bound = True
    return L


# ---------------------------------------------------------------- communicators
class TorchComm:
    """Collectives of one process group (NCCL on GPUs; gloo works for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce(self, t, op: str):
        d = self.dist
        self.dist.all_reduce(t, op={"min": d.ReduceOp.MIN, "max": d.ReduceOp.MAX, "sum": d.ReduceOp.SUM}[op],
                             group=self.group)

    def allgather_into(self, out, t):
        self.dist.all_gather_into_tensor(out, t, group=self.group)

    def alltoall(self, out, inp, out_splits, in_splits):
        self.dist.all_to_all_single(out, inp, list(out_splits), list(in_splits), group=self.group)

    def sizes(self, n: int, device):
        import torch
        t = torch.tensor([n], dtype=torch.int64, device=device)
        out = torch.empty(self.size, dtype=torch.int64, device=device)
        self.allgather_into(out, t)
        return [int(v) for v in out.cpu()]


class LoopbackHub:
    """Shared state of R in-process virtual ranks (threads)."""

    def __init__(self, R: int):
        self.R = R
        self.barrier = threading.Barrier(R)
        self.slots = [None] * R


class LoopbackComm:
    """R ranks as threads of one process: each posts its (stream-synchronised)
    tensor, every rank combines the posts on its own stream, then all wait until
    every copy is done before a post may be reused."""

    def __init__(self, hub: LoopbackHub, rank: int):
        self.hub, self.rank, self.size = hub, rank, hub.R

    def _exchange(self, v):
        import torch
        torch.cuda.current_stream().synchronize()
        self.hub.slots[self.rank] = v
        self.hub.barrier.wait()
        allv = list(self.hub.slots)
        return allv

    def _done(self):
        import torch
        torch.cuda.current_stream().synchronize()
        self.hub.barrier.wait()

    def allreduce(self, t, op: str):
        import torch
        allv = self._exchange(t)
        res = allv[0].clone()
        for v in allv[1:]:
            res = torch.minimum(res, v) if op == "min" else torch.maximum(res, v) if op == "max" else res + v
        self._done()
        t.copy_(res)

    def allgather_into(self, out, t):
        import torch
        allv = self._exchange(t)
        out.copy_(torch.cat(allv))
        self._done()

    def alltoall(self, out, inp, out_splits, in_splits):
        import torch
        allv = self._exchange((inp, list(in_splits)))
        pieces = []
        for q in range(self.size):
            src, sp = allv[q]
            o = sum(sp[: self.rank])
            pieces.append(src[o: o + sp[self.rank]])
        if out.numel():
            out.copy_(torch.cat(pieces))
        self._done()

    def sizes(self, n: int, device):
        allv = self._exchange(n)
        self._done()
        return [int(v) for v in allv]


# ---------------------------------------------------------------- the sort
class ShardInfo:
    """This rank's part of the global result: ``offset`` of its slice in the global
    output, its bucket range [jlo, jhi), and (with ``log=True``) its node records."""

    def __init__(self):
        self.offset = 0
        self.jlo = self.jhi = 0
        self.nodes = None
        self.level1_b = self.level1_h = None


def sort_sharded(x, comm, *, tau: int = 64, seed: int = 0, sample_all: bool = False, log: bool = False,
                 node_capacity=None, stream=None):
    """Sort the global array whose shard on this rank is ``x`` (1-D CUDA float64 /
    uint64, contiguous).  Returns ``(out, ShardInfo)``: ``out`` is this rank's slice
    of the sorted global array, starting at ``info.offset``."""
    import numpy as np
    import torch

    L = _bind()
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dim() != 1 or not x.is_contiguous():
        raise TypeError("x must be a contiguous 1-D CUDA tensor (no CPU fallback)")
    kt = {torch.float64: KEY_F64, torch.uint64: KEY_U64}.get(x.dtype)
    if kt is None:
        raise TypeError(f"keys must be float64 or uint64, got {x.dtype}")
    dev = x.device
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(s.cuda_stream)
    R, rank = comm.size, comm.rank
    n = x.numel()
    sizes = comm.sizes(n, dev)
    N = sum(sizes)
    offset = sum(sizes[:rank])
    info = ShardInfo()
    if N < 2 or N >= 2 ** 32:
        raise ValueError("the global array must hold 2 <= N < 2^32 keys")
    state = torch.empty(L.pcf_shard_state_bytes(N, R), dtype=torch.uint8, device=dev)
    sh = ShardC(N, offset, R, rank, state.data_ptr(), state.numel())
    shp = ctypes.byref(sh)
    views = (ctypes.c_void_p * 4)()
    vsz = (ctypes.c_uint64 * 4)()
    _check(L.pcf_shard_views(shp, views, vsz))

    def view(i, dtype, elem):
        o = views[i] - state.data_ptr()
        return state[o: o + vsz[i] * elem].view(dtype)

    mm, cnt, hloc, hall = view(0, torch.int64, 8), view(1, torch.int32, 4), view(2, torch.int32, 4), \
        view(3, torch.int32, 4)
    flags = FLAG_SAMPLE_ALL if sample_all else 0
    p = make_params(tau, seed, flags)
    pp = ctypes.cast(ctypes.byref(p), ctypes.c_void_p)
    xp = ctypes.c_void_p(x.data_ptr())
    with torch.cuda.stream(s):
        # 1. extremes of the global level-1 node
        _check(L.pcf_shard_minmax(xp, n, kt, shp, sp))
        comm.allreduce(mm[0:1], "min")
        comm.allreduce(mm[1:2], "max")
        comm.allreduce(mm[2:3], "max")
        # 2. the single-GPU sample, drawn where it lives; counts per bin
        _check(L.pcf_shard_counts(xp, n, kt, shp, pp, sp))
        comm.allreduce(cnt, "sum")   # u32 counts summed as int32: identical bits mod 2^32
        # 3. bucket histograms
        _check(L.pcf_shard_histogram(xp, n, kt, shp, pp, sp))
        comm.allgather_into(hall, hloc)
        # 4. bucket ranges -> ranks; keys grouped by destination, in input order
        grouped = torch.empty_like(x)
        send = (ctypes.c_uint64 * R)()
        recv = (ctypes.c_uint64 * R)()
        rng = (ctypes.c_uint64 * 4)()
        _check(L.pcf_shard_partition(xp, n, kt, shp, ctypes.c_void_p(grouped.data_ptr()), send, recv, rng, sp))
        m = int(rng[1])
        info.offset, info.jlo, info.jhi = int(rng[0]), int(rng[2]), int(rng[3])
        mine = torch.empty(m, dtype=x.dtype, device=dev)
        comm.alltoall(mine.view(torch.int64), grouped.view(torch.int64), [int(v) for v in recv],
                      [int(v) for v in send])
        del grouped
        # 5. the rest of Alg. 1 for this rank's buckets, at their global offset
        out = torch.empty(m, dtype=x.dtype, device=dev)
        ws = torch.empty(L.pcf_shard_workspace_bytes(m, N), dtype=torch.uint8, device=dev)
        p.workspace, p.workspace_bytes = ws.data_ptr(), ws.numel()
        p.flags = flags | FLAG_SYNC
        keep = []
        if log:
            cap = node_capacity if node_capacity is not None else min(N, 12 * (N // max(tau, 1))) + 64
            recs = torch.zeros(cap * 9, dtype=torch.int64, device=dev)
            cntl = torch.zeros(1, dtype=torch.int64, device=dev)
            l1 = int(lib().pcf_level1_entries(N, None))
            b = torch.zeros(l1, dtype=torch.int32, device=dev)
            h = torch.zeros(l1, dtype=torch.int32, device=dev)
            pl = PassLog(recs.data_ptr(), cap, cntl.data_ptr(), b.data_ptr(), h.data_ptr(), l1)
            p.log = ctypes.pointer(pl)
            keep += [recs, cntl, b, h, pl]
        _check(L.pcf_shard_sort_range(ctypes.c_void_p(mine.data_ptr()), ctypes.c_void_p(out.data_ptr()), m, kt, shp,
                                      rng, pp, sp))
    if log:
        k = int(cntl.item())
        arr = recs.view(torch.uint8).cpu().numpy()[: k * 72]
        info.nodes = np.frombuffer(arr.tobytes(), dtype=NODE_DTYPE()).copy()
        if rank == 0:
            info.level1_b = b.cpu().numpy().view(np.uint32)
            info.level1_h = h.cpu().numpy().view(np.uint32)
    return out, info

