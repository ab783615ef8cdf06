"""Per-kernel-class device times of one build under environment variants
(development aid for tuning; each variant runs in its own process).

    python tools/knobs.py [n] [k] [mode] [kind] -- VAR=val,VAR2=val ...
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, sys, torch, numpy as np
sys.path.insert(0, sys.argv[1])
sys.path.insert(0, sys.argv[1] + "/tools")
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import _native, datagen
n, k, mode, kind = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
from adv import make
pts = make(kind, n, k)
d = torch.from_numpy(pts).cuda(); out = torch.empty_like(d); perm = torch.empty(n, dtype=torch.int32, device="cuda")
f = (lambda: kd.build_round_robin_cuda(d, out=out, perm=perm, check_finite=False)) if mode == "rr" else \
    (lambda: kd.build_widest_cuda(d, out=out, perm=perm, check_finite=False))
for _ in range(3): f()
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
_native.set_profile(True); f(); torch.cuda.synchronize()
cls = {c: round(v[1], 3) for c, v in _native.profile_kernels().items()}
print("RESULT " + json.dumps({"ms": round(min(ts), 3), "classes": cls}))
'''

if __name__ == "__main__":
    args = sys.argv[1:]
    sep = args.index("--") if "--" in args else len(args)
    pos, variants = args[:sep], args[sep + 1:] or [""]
    n = pos[0] if len(pos) > 0 else "100000000"
    k = pos[1] if len(pos) > 1 else "3"
    mode = pos[2] if len(pos) > 2 else "rr"
    kind = pos[3] if len(pos) > 3 else "uniform"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for v in variants:
        env = dict(os.environ)
        for kv in filter(None, v.split(",")):
            a, b = kv.split("=", 1)
            env[a] = b
        try:
            r = subprocess.run([sys.executable, "-c", CHILD, root, n, k, mode, kind], env=env, capture_output=True,
                               text=True, timeout=int(os.environ.get("KNOBS_TIMEOUT", "180")))
        except subprocess.TimeoutExpired:
            print(json.dumps({"variant": v or "default", "n": int(n), "mode": mode, "kind": kind, "error": "timeout"}),
                  flush=True)
            continue
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        res = json.loads(line[0][7:]) if line else {"error": (r.stderr or r.stdout)[-400:]}
        print(json.dumps({"variant": v or "default", "n": int(n), "k": int(k), "mode": mode, "kind": kind, **res}),
              flush=True)
