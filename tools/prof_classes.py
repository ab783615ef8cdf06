"""Per-kernel-class device time of one build (lbkd_profile_kernel), both algorithms."""
import sys
import torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import _native, datagen

def run(n, k, mode="rr", kind="uniform", algo="select"):
    pts = datagen.make(kind, n, k, seed=0)
    d = torch.from_numpy(pts).cuda()
    out = torch.empty_like(d); perm = torch.empty(n, dtype=torch.int32, device="cuda")
    _native.set_algorithm(algo)
    f = (lambda: kd.build_round_robin_cuda(d, out=out, perm=perm, check_finite=False)) if mode == "rr" else \
        (lambda: kd.build_widest_cuda(d, out=out, perm=perm, check_finite=False))
    f(); f()
    _native.set_profile(True)
    f()
    torch.cuda.synchronize()
    prof = _native.profile_kernels()
    _native.set_profile(False)
    tot = sum(v[1] for v in prof.values())
    print(f"== {mode} {kind} n={n} k={k} algo={algo}: sum of kernel times {tot:.2f} ms")
    for name, (cnt, ms, by) in sorted(prof.items(), key=lambda x: -x[1][1]):
        print(f"   {name:10s} n={cnt:4d} {ms:8.3f} ms  {by/1e9:8.2f} GB  {by/ms/1e6 if ms else 0:8.1f} GB/s")

if __name__ == "__main__":
    run(10**8, 3)
    run(10**8, 3, algo="sort")
    run(10**8, 3, "widest", "clustered")
    run(10**8, 3, "widest", "clustered", algo="sort")
