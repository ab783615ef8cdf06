"""Multi-GPU round-robin build: one process per GPU.

The path shards naturally: after level t every level-t subtree is
independent (a stable sort restricted to a subset keeps that subset's
order), and in the in-order working layout each subtree is one contiguous
range of every SoA array.  With G = 2^t ranks the top levels are split by
RECURSIVE HALVING instead of running on rank 0 alone:

    step i = 0 .. t-1: every rank r that holds a level-i subtree (r a
    multiple of h = G >> i; rank 0 starts with the whole input) builds ONE
    level of it with lbkd_build_rr_split -- its node goes to the output, its
    points land in a fresh buffer in in-order layout, left child first --
    keeps the left child where it is and ships the right child's points (k
    coordinate arrays + index array, in the order the reference's sort leaves
    them) to rank r + h/2.  No copies besides the level's own partition: the
    packed buffers ARE the working sets (split and sub use them in place).

Then every rank finishes its level-t subtree (lbkd_build_rr_sub) with the
GLOBAL tree geometry (global node ids, pivot offsets, in-order positions),
so the result is bit-identical to the single-GPU build, and sends its nodes
back to rank 0: one contiguous level-order range per level of its subtree,
plus the single nodes it placed while splitting.  The critical path is
level 0 on N points + level 1 on N/2 + ... instead of t levels on N.

Transport: device tensors through the process group (NCCL over NVLink /
NVSwitch), or, for a gloo group (CPU tests, several ranks sharing one GPU),
the same messages staged through host memory.  The exchange logic is
independent of the device kernels (``ops`` is injectable), which is what the
CPU gloo tests exercise with fakes; tests/test_gpu_multiproc.py runs the
real kernels in two processes.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

from . import treemath


def ceil4(x: int) -> int:
    """Array stride of the packed buffers: whole 16-byte rows."""
    return (x + 3) & ~3


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


def split_plan(world: int):
    """Recursive halving: per step i the (holder, partner, level, index) of
    every split.  Holder r splits its level-i subtree j = r >> (t - i) and
    sends the right child (index 2j + 1) to partner r + (G >> (i + 1))."""
    t = top_levels_for(world)
    steps = []
    for i in range(t):
        h = world >> i
        steps.append([(r, r + h // 2, i, r >> (t - i)) for r in range(0, world, h)])
    return steps


def placed_nodes(world: int, rank: int):
    """The single nodes rank `rank` places while splitting (level i, node)."""
    return [(i, (1 << i) - 1 + j) for step in split_plan(world) for (r, _, i, j) in step if r == rank]


class CudaOps:
    """The device side: the C-ABI calls on torch CUDA tensors."""

    def __init__(self, device: int):
        from . import _native

        self.native = _native
        self.lib = _native.load()
        self.device = device

    def _stream(self, stream):
        import torch

        s = stream or torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def build_top(self, points, top, out, perm, sub, sub_stride, stream=None):
        n, k = points.shape
        ctx = self.native.context(self.device)
        rc = self.lib.lbkd_build_rr_top(ctx, points.data_ptr(), n, k, top, out.data_ptr(), perm.data_ptr(),
                                        sub.data_ptr(), sub_stride, self._stream(stream))
        self.native.check(rc, "lbkd_build_rr_top")

    def build_split(self, points, sub, stride, n, k, level, j, out, perm, nxt, stream=None):
        """One level of subtree (level, j): from ``points`` (raw, level 0) or
        the packed ``sub``; ``nxt`` receives the children in in-order layout
        (same stride)."""
        ctx = self.native.context(self.device)
        rc = self.lib.lbkd_build_rr_split(ctx, points.data_ptr() if points is not None else None,
                                          sub.data_ptr() if sub is not None else None, stride, n, k, level, j,
                                          out.data_ptr(), perm.data_ptr(), nxt.data_ptr(), self._stream(stream))
        self.native.check(rc, "lbkd_build_rr_split")

    def build_sub(self, sub, sub_stride, n, k, top, j, out, perm, stream=None):
        ctx = self.native.context(self.device)
        rc = self.lib.lbkd_build_rr_sub(ctx, sub.data_ptr(), sub_stride, n, k, top, j, out.data_ptr(),
                                        perm.data_ptr(), self._stream(stream))
        self.native.check(rc, "lbkd_build_rr_sub")


class _Transport:
    """Point-to-point messages of device tensors: direct for NCCL; staged
    through host memory for gloo (which only moves CPU tensors)."""

    def __init__(self, group, device):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.host = dist.get_backend(group) == "gloo" and device.type == "cuda"

    def exchange(self, sends, recvs):
        """sends: [(tensor, peer)], recvs: [(tensor, peer)] -- all posted at
        once, then waited for; received data lands in the given tensors."""
        dist = self.dist
        ops = []
        staged = []
        for t, peer in sends:
            ops.append(dist.P2POp(dist.isend, t.cpu() if self.host else t, peer, self.group))
        for t, peer in recvs:
            buf = t.new_empty(t.shape, device="cpu") if self.host else t
            ops.append(dist.P2POp(dist.irecv, buf, peer, self.group))
            if self.host:
                staged.append((t, buf))
        if ops:
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        for t, buf in staged:
            t.copy_(buf)


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
    t = top_levels_for(world)
    dev = device if device is not None else (points.device if points is not None else torch.device("cpu"))
    if ops is None:
        ops = CudaOps(dev.index if dev.type == "cuda" else 0)
    tr = _Transport(group, dev)
    bufs = buffers if buffers is not None else {}

    def buf(name, shape, dtype):
        b = bufs.get(name)
        if b is None or b.shape != torch.Size(shape) or b.dtype != dtype:
            b = torch.empty(shape, dtype=dtype, device=dev)
            bufs[name] = b
        return b

    out = buf("out", (n, k), torch.float32)
    perm = buf("perm", (n,), torch.int32)
    if world == 1:
        from . import builder

        builder.build_round_robin_cuda(points, out=out, perm=perm, check_finite=False)
        return out, perm
    # ---- recursive halving of the top t levels
    cur = None          # the subtree this rank holds: k + 1 arrays `stride` words apart
    cur_level, cur_j, stride = 0, 0, ceil4(n)
    for i, step in enumerate(split_plan(world)):
        for (r, partner, level, j) in step:
            s = (1 << level) - 1 + j
            lc = 2 * s + 1
            lsize = treemath.subtree_size(lc, n) if lc < n else 0
            rsize = treemath.subtree_size(lc + 1, n) if lc + 1 < n else 0
            if rank == r:
                nxt = buf(f"split{i}", ((k + 1) * stride,), torch.int32)
                ops.build_split(points if level == 0 else None, cur, stride, n, k, level, j, out, perm, nxt)
                # the right child sits after the node's slot in every array
                sends = [(nxt[c * stride + lsize + 1:c * stride + lsize + 1 + rsize], partner) for c in range(k + 1)]
                tr.exchange(sends, [])
                cur, cur_level, cur_j = nxt, level + 1, 2 * j  # the left child stays in place
            elif rank == partner:
                rstride = ceil4(rsize)
                recv = buf(f"recv{i}", ((k + 1) * rstride,), torch.int32)
                tr.exchange([], [(recv[c * rstride:c * rstride + rsize], r) for c in range(k + 1)])
                cur, cur_level, cur_j, stride = recv, level + 1, 2 * j + 1, rstride
    # ---- every rank finishes its level-t subtree
    assert cur_level == t and cur_j == rank
    ops.build_sub(cur, stride, n, k, t, rank, out, perm)
    # ---- gather at rank 0: subtree node ranges + the single split nodes
    if rank == 0:
        recvs = []
        for peer in range(1, world):
            for first, cnt in node_ranges(n, t, peer):
                recvs.append((out[first:first + cnt], peer))
                recvs.append((perm[first:first + cnt], peer))
            for _, node in placed_nodes(world, peer):
                recvs.append((out[node:node + 1], peer))
                recvs.append((perm[node:node + 1], peer))
        tr.exchange([], recvs)
        return out, perm
    sends = []
    for first, cnt in node_ranges(n, t, rank):
        sends.append((out[first:first + cnt], 0))
        sends.append((perm[first:first + cnt], 0))
    for _, node in placed_nodes(world, rank):
        sends.append((out[node:node + 1], 0))
        sends.append((perm[node:node + 1], 0))
    tr.exchange(sends, [])
    return None, None


def serial_sharded_build(points, n: int, k: int, world: int, ops=None, out=None, perm=None, timer=None):
    """The whole protocol of build_round_robin_sharded run rank by rank in
    ONE process on one device (no transport): the same kernels and buffers,
    so the result must equal the single-GPU build.  ``timer(label, fn)`` may
    wrap every device call (tools/big_build.py times each piece to project
    the multi-GPU critical path).  Returns (out, perm)."""
    import torch

    dev = points.device
    t = top_levels_for(world)
    if ops is None:
        ops = CudaOps(dev.index if dev.type == "cuda" else 0)
    if out is None:
        out = torch.empty((n, k), dtype=torch.float32, device=dev)
    if perm is None:
        perm = torch.empty(n, dtype=torch.int32, device=dev)
    run = timer or (lambda label, fn: fn())
    held = {0: (None, ceil4(n))}  # rank -> (its subtree's buffer, stride)
    for i, step in enumerate(split_plan(world)):
        for (r, partner, level, j) in step:
            s = (1 << level) - 1 + j
            lc = 2 * s + 1
            lsize = treemath.subtree_size(lc, n) if lc < n else 0
            rsize = treemath.subtree_size(lc + 1, n) if lc + 1 < n else 0
            cur, stride = held[r]
            nxt = torch.empty((k + 1) * stride, dtype=torch.int32, device=dev)
            run(f"split{i}/r{r}", lambda: ops.build_split(points if level == 0 else None, cur, stride, n, k, level, j,
                                                          out, perm, nxt))
            rstride = ceil4(rsize)
            right = torch.empty((k + 1) * rstride, dtype=torch.int32, device=dev)
            for c in range(k + 1):  # (the transfer to the partner rank)
                right[c * rstride:c * rstride + rsize].copy_(nxt[c * stride + lsize + 1:c * stride + lsize + 1 + rsize])
            held[r] = (nxt, stride)
            held[partner] = (right, rstride)
    for r in range(world):
        sub, stride = held[r]
        run(f"sub/r{r}", lambda: ops.build_sub(sub, stride, n, k, t, r, out, perm))
    return out, perm
