"""One warm-up build + one build (for ncu launch lists / captures)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
sys.path.insert(0, __file__.rsplit('/', 1)[0])
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import datagen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**8
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
mode = sys.argv[3] if len(sys.argv) > 3 else "rr"
kind = sys.argv[4] if len(sys.argv) > 4 else "uniform"
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
from adv import make  # noqa: E402

pts = make(kind, n, k)
d = torch.from_numpy(pts).cuda()
out = torch.empty_like(d); perm = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(reps):
    if mode == "rr":
        kd.build_round_robin_cuda(d, out=out, perm=perm)
    else:
        kd.build_widest_cuda(d, out=out, perm=perm)
torch.cuda.synchronize()
print("launches per build:", kd.builder.last_launch_count(0))
