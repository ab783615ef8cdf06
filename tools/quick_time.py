"""Quick device-side timing of builds (development aid)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import datagen

def t(n, k, mode="rr", kind="uniform", reps=5):
    pts = datagen.make(kind, n, k, seed=0)
    d = torch.from_numpy(pts).cuda()
    out = torch.empty_like(d); perm = torch.empty(n, dtype=torch.int32, device="cuda")
    f = (lambda: kd.build_round_robin_cuda(d, out=out, perm=perm, check_finite=False)) if mode == "rr" else \
        (lambda: kd.build_widest_cuda(d, out=out, perm=perm, check_finite=False))
    for _ in range(2): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    ms = min(ts)
    print(f"{mode} {kind} n={n} k={k}: {ms:.3f} ms  {n/ms/1e3:.1f} Mpts/s  (all {['%.2f'%x for x in ts]})", flush=True)

if __name__ == "__main__":
    for n in [10**6, 10**7, 10**8]:
        t(n, 3)
    t(10**8, 2); t(10**7, 4)
    t(10**8, 3, "widest", "clustered")
    t(10**8, 3, "rr", "clustered")
