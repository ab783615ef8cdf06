"""Config 4 (BASELINE.json): float3 clustered N=1B round-robin, on ONE B200.

1. The single-GPU build of all 1B points (CUDA events, warm-up + reps).
2. lbkd_check_valid of the result on the device (verify.py:195-245).
3. The sharded protocol of multigpu.build_round_robin_sharded for G = 2, 4,
   8 run rank by rank on this one GPU (multigpu.serial_sharded_build):
   recursive halving of the top log2 G levels (lbkd_build_rr_top with one
   level, then lbkd_build_rr_split), then lbkd_build_rr_sub for every
   subtree, each piece timed alone.  The result must equal the single-GPU
   build bit for bit, and sum over steps of the slowest holder + the slowest
   subtree is the device time a G-GPU run would need before its NVLink
   exchanges -- reported as a projection, not a measured scaling.

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
out2 = torch.empty_like(d)
perm2 = torch.empty_like(perm)
shard = {}
for G in (2, 4, 8):
    best = None
    for _ in range(2):
        times = {}

        def timer(label, fn):
            a, b = ev(), ev()
            a.record()
            fn()
            b.record()
            times[label] = (a, b)

        multigpu.serial_sharded_build(d, n, k, G, ops=ops, out=out2, perm=perm2, timer=timer)
        torch.cuda.synchronize()
        ms = {lab: x.elapsed_time(y) for lab, (x, y) in times.items()}
        # critical path: each halving step waits for its slowest holder, then
        # the slowest subtree (exchange time not included)
        steps = sorted({lab.split("/")[0] for lab in ms if lab.startswith("split")})
        split_ms = [max(v for lab, v in ms.items() if lab.startswith(s + "/")) for s in steps]
        sub_ms = [ms[f"sub/r{r}"] for r in range(G)]
        crit = sum(split_ms) + max(sub_ms)
        if best is None or crit < best[0]:
            best = (crit, split_ms, sub_ms)
    same = bool(torch.equal(out2, out) and torch.equal(perm2, perm))
    crit, split_ms, sub_ms = best
    t = multigpu.top_levels_for(G)
    moved = sum(sh.size for sh in multigpu.shard_layout(n, t)[1:])
    shard[G] = {"split_step_ms": [round(x, 2) for x in split_ms], "sub_ms": [round(x, 2) for x in sub_ms],
                "critical_path_ms_before_exchange": round(crit, 2),
                "points_shipped_in_halving": sum(multigpu.shard_layout(n, t)[j].size for j in range(1, G)),
                "bytes_back_to_rank0": moved * 4 * (k + 1),
                "bit_identical_to_single_gpu": same}
    print(json.dumps({"G": G, **shard[G]}), flush=True)
res["sharded_on_one_gpu_recursive_halving"] = shard
print(json.dumps(res))
