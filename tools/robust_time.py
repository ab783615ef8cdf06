"""Build times on adversarial inputs (robustness of the selection path)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import datagen
from oracle import oracle

def run(name, pts, check=False, mode="rr"):
    d = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32)).cuda()
    f = (lambda: kd.build_round_robin_cuda(d)) if mode == "rr" else (lambda: kd.build_widest_cuda(d))
    r = f(); torch.cuda.synchronize()
    t0 = time.time(); r = f(); torch.cuda.synchronize(); dt = time.time() - t0
    ok = ""
    if check:
        want = oracle.build_rr(pts) if mode == "rr" else oracle.build_widest(pts)[0]
        ok = "exact" if np.array_equal(r[1].cpu().numpy().view(np.uint32), want) else "MISMATCH"
    print(f"{name:40s} n={len(pts):>11,} {mode}: {dt*1e3:9.2f} ms {ok}", flush=True)

n = 10_000_000
run("all points identical", np.full((n, 3), 0.25, np.float32), check=True)
run("ties: 64 values per axis", datagen.ties(n, 3, seed=1), check=True)
run("sorted along x", np.sort(datagen.uniform(n, 3, seed=2), axis=0), check=True)
run("one axis constant", np.c_[datagen.uniform(n, 2, seed=3), np.zeros(n, np.float32)], check=True)
run("huge range (1e-30..1e30)", (10.0 ** np.random.default_rng(4).uniform(-30, 30, (n, 3))).astype(np.float32), check=True)
run("clustered", datagen.clustered(n, 3, seed=5), check=True)
run("all points identical", np.full((n, 3), 0.25, np.float32), check=True, mode="widest")
run("ties: 64 values per axis", datagen.ties(n, 3, seed=1), check=True, mode="widest")
N = 100_000_000
run("clustered", datagen.clustered(N, 3, seed=0))
run("ties: 64 values per axis", datagen.ties(N, 3, seed=1))
