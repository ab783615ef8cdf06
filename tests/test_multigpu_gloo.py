"""Multi-process (gloo, CPU) tests of the sharded build's host logic:
shard layout, node ranges, and the rank0 -> rank j -> rank0 exchange.

The device kernels are replaced by fakes that stamp every value with its
origin, so the test proves each subtree's points reach the right rank and
every node comes back to its level-order slot exactly once.  The device
path itself is checked bit-exact on one GPU in test_gpu_parity.py.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_00120_b200 import multigpu, treemath


def test_layout_and_ranges_partition_the_tree():
    for n in (15, 16, 100, 1000, 4097, 123457, 10**6):
        for world in (2, 4, 8):
            top = multigpu.top_levels_for(world)
            if (1 << (top + 1)) - 1 > n:
                continue
            lay = multigpu.shard_layout(n, top)
            F = (1 << top) - 1
            assert sum(s.size for s in lay) == n - F
            off = 0
            for s in lay:
                assert s.offset == off
                off += s.size
            seen = np.zeros(n, dtype=np.int32)
            seen[:F] += 1
            for s in lay:
                cnt = 0
                for first, c in multigpu.node_ranges(n, top, s.index):
                    seen[first:first + c] += 1
                    cnt += c
                assert cnt == s.size == treemath.subtree_size(s.node, n)
            assert np.all(seen == 1), (n, world)
    with pytest.raises(ValueError):
        multigpu.top_levels_for(3)


def _stamp(level, j, c, i):
    return (level * 15485863 + j * 7919 + c * 104729 + i * 31) % 1000003


class FakeOps:
    """Stamps every point value with (level, subtree, array, position) and
    every node with its own id, and checks each stamp where it is consumed
    (the real layout: split writes the children in in-order layout, left
    child first, one slot for the node, then the right child)."""

    def __init__(self, rank):
        self.rank = rank

    def _fill(self, buf, stride, k, level, j, size, off=0):
        i = torch.arange(size)
        for c in range(k + 1):
            buf[c * stride + off:c * stride + off + size] = _stamp(level, j, c, i)

    def _place(self, out, perm, node):
        perm[node] = node
        out[node] = float(node)

    def _check(self, sub, stride, n, k, level, j):
        size = treemath.subtree_size((1 << level) - 1 + j, n)
        i = torch.arange(size)
        for c in range(k + 1):
            got = sub[c * stride:c * stride + size]
            assert torch.equal(got, _stamp(level, j, c, i).to(torch.int32)), (self.rank, level, j, c)

    def build_split(self, points, sub, stride, n, k, level, j, out, perm, nxt):
        assert stride % 4 == 0
        if level == 0:
            assert points is not None and stride == multigpu.ceil4(n)
        else:
            self._check(sub, stride, n, k, level, j)
        s = (1 << level) - 1 + j
        self._place(out, perm, s)
        lc = 2 * s + 1
        lsize = treemath.subtree_size(lc, n) if lc < n else 0
        if lc < n:
            self._fill(nxt, stride, k, level + 1, 2 * j, lsize)
        if lc + 1 < n:
            self._fill(nxt, stride, k, level + 1, 2 * j + 1, treemath.subtree_size(lc + 1, n), off=lsize + 1)

    def build_sub(self, sub, stride, n, k, top, j, out, perm):
        self._check(sub, stride, n, k, top, j)
        for first, cnt in multigpu.node_ranges(n, top, j):
            ids = torch.arange(first, first + cnt)
            perm[first:first + cnt] = ids.to(torch.int32)
            out[first:first + cnt] = ids.to(torch.float32)[:, None]


def test_split_plan_covers_every_top_node_once():
    for world in (2, 4, 8, 16):
        t = multigpu.top_levels_for(world)
        placed = sorted(node for r in range(world) for _, node in multigpu.placed_nodes(world, r))
        assert placed == list(range((1 << t) - 1)), world
        for i, step in enumerate(multigpu.split_plan(world)):
            assert len(step) == 1 << i
            # a holder at step i received its subtree at an earlier step (or is rank 0)
            for r, partner, level, j in step:
                assert level == i and partner == r + (world >> (i + 1))
                assert r >> (t - i) == j


def _worker(rank, world, port, n, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = torch.zeros((n, k), dtype=torch.float32) if rank == 0 else None
        out, perm = multigpu.build_round_robin_sharded(pts, n, k, ops=FakeOps(rank), device=torch.device("cpu"))
        if rank == 0:
            ok = torch.equal(perm, torch.arange(n, dtype=torch.int32)) and torch.equal(
                out, torch.arange(n, dtype=torch.float32)[:, None].expand(n, k))
            q.put(bool(ok))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,n,k", [(2, 1001, 3), (4, 40000, 2), (2, 65537, 4), (8, 100003, 3)])
def test_sharded_exchange_gloo(world, n, k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
