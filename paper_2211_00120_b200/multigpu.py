"""Multi-GPU round-robin build: one process per GPU.

The path shards naturally after one exchange step.  Rank 0 holds the input
and builds the top ``t = log2(G)`` levels; after them every level-t subtree
is independent (a stable sort restricted to a subset keeps that subset's
order), and in the in-order working layout each subtree is one contiguous
range of every SoA array.  So:

1. rank 0: ``lbkd_build_rr_top`` -- levels 0..t-1, nodes written at their
   level-order slots, subtree j's points packed at offset
   ``segment_begin(F(t)+j) - F(t)`` (k coordinate arrays + index array);
2. rank 0 -> rank j: k+1 contiguous slices (NCCL send/recv over NVLink);
3. every rank j: ``lbkd_build_rr_sub`` -- the remaining levels of subtree j
   with the GLOBAL tree geometry (global node ids, pivot offsets, in-order
   positions), so the result is bit-identical to the single-GPU build;
4. rank j -> rank 0: subtree j's nodes, one contiguous range per level.

The exchange logic is independent of the device kernels (``ops`` is
injectable), which is what the gloo tests on CPU exercise.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import treemath


def top_levels_for(world: int) -> int:
    if world < 1 or world & (world - 1):
        raise ValueError("the sharded build needs a power-of-two number of ranks")
    return world.bit_length() - 1


@dataclass(frozen=True)
class Shard:
    index: int      # subtree j at level `top`
    node: int       # its root node F(top) + j
    offset: int     # packed offset in the send buffer
    size: int       # points in the subtree


def shard_layout(n: int, top: int):
    """The 2^top level-`top` subtrees of an n-point tree, in node order."""
    F = (1 << top) - 1
    out = []
    for j in range(1 << top):
        s = F + j
        out.append(Shard(j, s, treemath.segment_begin(s, n) - F, treemath.subtree_size(s, n)))
    return out


def node_ranges(n: int, top: int, j: int):
    """Level-order node ranges (first, count) owned by subtree j: at level l
    its nodes are F(l) + [j, j+1) * 2^(l-top), clipped to n."""
    L = treemath.num_levels(n)
    out = []
    for l in range(top, L):
        first = (1 << l) - 1 + (j << (l - top))
        last = min(first + (1 << (l - top)), n)
        if first < last:
            out.append((first, last - first))
    return out


class CudaOps:
    """The device side: the C-ABI calls on torch CUDA tensors."""

    def __init__(self, device: int):
        from . import _native

        self.native = _native
        self.lib = _native.load()
        self.device = device

    def build_top(self, points, top, out, perm, sub, sub_stride, stream=None):
        import torch

        n, k = points.shape
        ctx = self.native.context(self.device)
        s = stream or torch.cuda.current_stream()
        rc = self.lib.lbkd_build_rr_top(ctx, points.data_ptr(), n, k, top, out.data_ptr(), perm.data_ptr(),
                                        sub.data_ptr(), sub_stride, ctypes.c_void_p(s.cuda_stream))
        self.native.check(rc, "lbkd_build_rr_top")

    def build_sub(self, sub, sub_stride, n, k, top, j, out, perm, stream=None):
        import torch

        ctx = self.native.context(self.device)
        s = stream or torch.cuda.current_stream()
        rc = self.lib.lbkd_build_rr_sub(ctx, sub.data_ptr(), sub_stride, n, k, top, j, out.data_ptr(),
                                        perm.data_ptr(), ctypes.c_void_p(s.cuda_stream))
        self.native.check(rc, "lbkd_build_rr_sub")


def build_round_robin_sharded(points, n: int, k: int, group=None, ops=None, device=None, buffers=None):
    """One n-point round-robin build spread over the ranks of `group`.

    ``points`` (n, k) float32 is only read on rank 0 (may be None elsewhere).
    Returns (out, perm) on rank 0 -- the complete level-order points and
    permutation -- and (None, None) on the other ranks.
    """
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    top = top_levels_for(world)
    dev = device if device is not None else (points.device if points is not None else torch.device("cpu"))
    if ops is None:
        ops = CudaOps(dev.index if dev.type == "cuda" else 0)
    layout = shard_layout(n, top)
    bufs = buffers if buffers is not None else {}

    def buf(name, shape, dtype):
        t = bufs.get(name)
        if t is None or t.shape != torch.Size(shape) or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, device=dev)
            bufs[name] = t
        return t

    out = buf("out", (n, k), torch.float32)
    perm = buf("perm", (n,), torch.int32)
    if rank == 0:
        sub = buf("sub", ((k + 1) * n,), torch.int32)
        ops.build_top(points, top, out, perm, sub, n)
        ops_list = []
        for sh in layout[1:]:
            for c in range(k + 1):
                base = c * n + sh.offset
                ops_list.append(dist.P2POp(dist.isend, sub[base:base + sh.size], sh.index, group))
        reqs = dist.batch_isend_irecv(ops_list) if ops_list else []
        ops.build_sub(sub, n, n, k, top, 0, out, perm)
        for r in reqs:
            r.wait()
        recv = []
        for sh in layout[1:]:
            for first, cnt in node_ranges(n, top, sh.index):
                recv.append(dist.P2POp(dist.irecv, out[first:first + cnt], sh.index, group))
                recv.append(dist.P2POp(dist.irecv, perm[first:first + cnt], sh.index, group))
        for r in (dist.batch_isend_irecv(recv) if recv else []):
            r.wait()
        return out, perm
    sh = layout[rank]
    sub = buf("sub", ((k + 1) * sh.size,), torch.int32)
    recv = [dist.P2POp(dist.irecv, sub[c * sh.size:(c + 1) * sh.size], 0, group) for c in range(k + 1)]
    for r in dist.batch_isend_irecv(recv):
        r.wait()
    ops.build_sub(sub, sh.size, n, k, top, sh.index, out, perm)
    send = []
    for first, cnt in node_ranges(n, top, sh.index):
        send.append(dist.P2POp(dist.isend, out[first:first + cnt], 0, group))
        send.append(dist.P2POp(dist.isend, perm[first:first + cnt], 0, group))
    for r in dist.batch_isend_irecv(send):
        r.wait()
    return None, None
