"""The sharded build (multigpu.build_round_robin_sharded)
with the REAL kernels in several processes: 2 and 4 ranks share the one GPU
of the test box, talk over a gloo process group (messages staged through host
memory -- the same exchange NCCL does device to device over NVLink), and the
result on rank 0 must equal the single-GPU build and the oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, k, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2211_00120_b200 import datagen, multigpu

        pts = torch.from_numpy(datagen.make(kind, n, k, seed=7)).cuda() if rank == 0 else None
        out, perm = multigpu.build_round_robin_sharded(pts, n, k, device=torch.device("cuda", 0))
        if rank == 0:
            import paper_2211_00120_b200 as kd
            from oracle import oracle

            ref_out, ref_perm = kd.build_round_robin_cuda(pts)
            p = perm.cpu().numpy().view(np.uint32)
            ok = (torch.equal(perm, ref_perm) and torch.equal(out.view(torch.int32), ref_out.view(torch.int32))
                  and np.array_equal(p, oracle.rec_build(pts.cpu().numpy())))
            q.put(bool(ok))
        torch.cuda.synchronize()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k,kind", [(2, 2_000_003, 3, "clustered"), (4, 1_000_000, 4, "uniform"),
                                            (2, 300_001, 2, "ties"), (8, 5_000_000, 3, "uniform")])
def test_sharded_build_real_kernels_multi_process(world, n, k, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, k, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
