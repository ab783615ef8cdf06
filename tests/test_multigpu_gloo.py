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


def _stamp(j, c, i):
    return (j * 7919 + c * 104729 + i * 31) % 1000003


class FakeOps:
    def __init__(self, rank):
        self.rank = rank

    def build_top(self, points, top, out, perm, sub, stride):
        n, k = points.shape
        F = (1 << top) - 1
        perm[:F] = torch.arange(F, dtype=torch.int32)
        out[:F] = torch.arange(F, dtype=torch.float32)[:, None]
        for sh in multigpu.shard_layout(n, top):
            i = torch.arange(sh.size)
            for c in range(k + 1):
                sub[c * stride + sh.offset: c * stride + sh.offset + sh.size] = _stamp(sh.index, c, i)

    def build_sub(self, sub, stride, n, k, top, j, out, perm):
        size = multigpu.shard_layout(n, top)[j].size
        i = torch.arange(size)
        for c in range(k + 1):
            got = sub[c * stride: c * stride + size]
            assert torch.equal(got, _stamp(j, c, i).to(torch.int32)), (self.rank, j, c)
        for first, cnt in multigpu.node_ranges(n, top, j):
            ids = torch.arange(first, first + cnt)
            perm[first:first + cnt] = ids.to(torch.int32)
            out[first:first + cnt] = ids.to(torch.float32)[:, None]


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


@pytest.mark.parametrize("world,n,k", [(2, 1001, 3), (4, 40000, 2), (2, 65537, 4)])
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
