"""Run one build (n, k, mode, kind) and compare with the oracle (debug aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import datagen
from oracle import oracle

n = int(sys.argv[1]); k = int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "rr"
kind = sys.argv[4] if len(sys.argv) > 4 else "uniform"
pts = datagen.make(kind, n, k, seed=0)
d = torch.from_numpy(pts).cuda()
if mode == "rr":
    out, perm = kd.build_round_robin_cuda(d)
    want = oracle.build_rr(pts)
else:
    out, perm, dims = kd.build_widest_cuda(d)
    want, wd = oracle.build_widest(pts)
got = perm.cpu().numpy().view(np.uint32)
bad = np.nonzero(got != want)[0]
print(f"n={n} k={k} {mode} {kind}: mismatches {len(bad)}", bad[:10], got[bad[:5]], want[bad[:5]])
