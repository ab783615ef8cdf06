"""Workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every build path at 200K points plus the query / verify kernels,
each result checked against the oracle so a silent corruption also fails.

    compute-sanitizer --tool memcheck python tools/sanitize.py [n]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import _native, datagen  # noqa: E402
from paper_2211_00120_b200.builder import build_round_robin_host, host_join  # noqa: E402
from paper_2211_00120_b200.verify import check_valid_cuda  # noqa: E402
from oracle import oracle  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
bad = 0


def check(name, got, want):
    global bad
    ok = np.array_equal(got, want)
    bad += not ok
    print(f"{name:40s} {'ok' if ok else 'MISMATCH'}", flush=True)


for kind, k in (("uniform", 3), ("ties", 2), ("clustered", 4), ("signed_zero", 3)):
    p = datagen.make(kind, n, k, seed=1)
    d = torch.from_numpy(p).cuda()
    out, perm = kd.build_round_robin_cuda(d)
    check(f"rr {kind} k{k}", perm.cpu().numpy().view(np.uint32), oracle.rec_build(p))
    assert check_valid_cuda(out) is None
    out, perm, dims = kd.build_widest_cuda(d)
    wp, wd = oracle.rec_build(p, widest=True)
    check(f"widest {kind} k{k}", perm.cpu().numpy().view(np.uint32), wp)
    check(f"widest dims {kind} k{k}", dims.cpu().numpy(), wd)
    q = torch.from_numpy(datagen.uniform(256, k, seed=2).astype(np.float64)).cuda()
    kd.knn_cuda(out, q, 8, split_dims=dims)
    kd.radius_cuda(out, q, 0.05, split_dims=dims)

# literal per-level radix sort path (decoupled lookback)
_native.set_algorithm("sort")
p = datagen.make("uniform", n, 3, seed=3)
_, perm = kd.build_round_robin_cuda(torch.from_numpy(p).cuda())
check("rr sort-path uniform k3", perm.cpu().numpy().view(np.uint32), oracle.rec_build(p))
_native.set_algorithm("select")

# in-CTA selection kernel for RR
_native.set_subtree_kernel("selection")
p = datagen.make("ties", n, 3, seed=4)
_, perm = kd.build_round_robin_cuda(torch.from_numpy(p).cuda())
check("rr selection-subtree ties k3", perm.cpu().numpy().view(np.uint32), oracle.rec_build(p))
_native.set_subtree_kernel("default")

# pipelined host builds
hp = datagen.make("clustered", n, 3, seed=5)
hin = torch.from_numpy(hp).pin_memory()
hout = torch.empty((n, 3), dtype=torch.float32).pin_memory()
hperm = torch.empty(n, dtype=torch.int32).pin_memory()
build_round_robin_host(hin, hout, hperm)
host_join()
check("rr host pipeline clustered k3", hperm.numpy().view(np.uint32), oracle.rec_build(hp))
torch.cuda.synchronize()
print("SANITIZE_WORKLOAD_DONE bad=%d" % bad, flush=True)
sys.exit(1 if bad else 0)
