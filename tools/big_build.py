"""Config 4 (BASELINE.json): float3 clustered N=1B round-robin, on ONE B200.

1. The single-GPU build of all 1B points (CUDA events, warm-up + reps).
2. lbkd_check_valid of the result on the device (verify.py:195-245).
3. The sharded decomposition of SURVEY.md §8(e) for G = 2, 4, 8, run on this
   one GPU: lbkd_build_rr_top (levels 0..log2 G - 1) then lbkd_build_rr_sub
   for every subtree j in turn, each timed alone.  The result must equal the
   single-GPU build bit for bit (the 1B check that needs no CPU oracle), and
   top + max_j sub is the device time a G-GPU run would need before its
   NVLink exchange -- reported as a projection, not a measured scaling.

Usage: python tools/big_build.py [n] [kind] [reps]   -> JSON on stdout
"""
import json
import sys
import time

import torch

sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import datagen, multigpu  # noqa: E402
from paper_2211_00120_b200.verify import check_valid_cuda  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**9
kind = sys.argv[2] if len(sys.argv) > 2 else "clustered"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
k = 3


def ev():
    return torch.cuda.Event(enable_timing=True)


t0 = time.time()
pts = datagen.make(kind, n, k, seed=0)
gen_s = time.time() - t0
d = torch.from_numpy(pts).cuda()
del pts
out = torch.empty_like(d)
perm = torch.empty(n, dtype=torch.int32, device="cuda")
kd.build_round_robin_cuda(d, out=out, perm=perm)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a, b = ev(), ev()
    a.record()
    kd.build_round_robin_cuda(d, out=out, perm=perm)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = min(ts)
wit = check_valid_cuda(out)
res = {"n": n, "k": k, "kind": kind, "gen_s": round(gen_s, 1), "build_ms": [round(x, 2) for x in ts],
       "mpts_per_s": round(n / ms / 1e3, 1), "check_valid": wit is None,
       "launches_per_build": kd.builder.last_launch_count(0),
       "mem_gb_peak": round(torch.cuda.max_memory_allocated() / 1e9, 1)}
print(json.dumps(res), flush=True)

ops = multigpu.CudaOps(0)
sub = torch.empty((k + 1) * n, dtype=torch.int32, device="cuda")
out2 = torch.empty_like(d)
perm2 = torch.empty_like(perm)
shard = {}
for G in (2, 4, 8):
    top = multigpu.top_levels_for(G)
    layout = multigpu.shard_layout(n, top)
    best = None
    for _ in range(2):
        a, b = ev(), ev()
        a.record()
        ops.build_top(d, top, out2, perm2, sub, n)
        b.record()
        subs = []
        for sh in layout:
            s0, s1 = ev(), ev()
            s0.record()
            ops.build_sub(sub[sh.offset:], n, n, k, top, sh.index, out2, perm2)
            s1.record()
            subs.append((s0, s1))
        torch.cuda.synchronize()
        top_ms = a.elapsed_time(b)
        sub_ms = [x.elapsed_time(y) for x, y in subs]
        if best is None or top_ms + max(sub_ms) < best[0] + max(best[1]):
            best = (top_ms, sub_ms)
    same = bool(torch.equal(out2, out) and torch.equal(perm2, perm))
    top_ms, sub_ms = best
    moved = sum(sh.size for sh in layout[1:])
    shard[G] = {"top_ms": round(top_ms, 2), "sub_ms": [round(x, 2) for x in sub_ms],
                "critical_path_ms": round(top_ms + max(sub_ms), 2),
                "points_moved_off_rank0": moved,
                "nvlink_bytes_each_way": moved * 4 * (k + 1),
                "bit_identical_to_single_gpu": same}
    print(json.dumps({"G": G, **shard[G]}), flush=True)
res["sharded_on_one_gpu"] = shard
print(json.dumps(res))
