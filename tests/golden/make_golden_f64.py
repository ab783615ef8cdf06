"""Golden hashes of the reference on float64 input (its own dtype).

Runs the reference (/root/reference, authoring container only) on the float64
generators of tests/golden_util.gen_f64 -- none of them float32-representable
-- and records sha256 of the output permutation (uint32) and split dims.

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden_f64.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
os.environ.setdefault("LBKD_BACKEND", "numba")

import lbkd  # noqa: E402  (the reference)

from golden_util import gen_f64  # noqa: E402

CASES = [
    ("uniform64", 1_000_000, 4, 0), ("uniform64", 200_000, 3, 1), ("uniform64", 65_537, 2, 2),
    ("ties64", 300_000, 3, 3), ("signed_zero64", 50_000, 3, 4), ("clustered64", 300_000, 3, 5),
    ("near64", 100_000, 3, 6), ("range64", 100_000, 3, 7), ("mixed64", 100_000, 3, 8),
    ("uniform64", 3_000, 3, 9), ("ties64", 4_000, 2, 10),
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    for kind, n, k, seed in CASES:
        pts = gen_f64(kind, n, k, seed)
        for mode in ("rr", "widest"):
            t0 = time.time()
            t = lbkd.build_round_robin(pts, k) if mode == "rr" else lbkd.build_widest(pts, k)
            dt = time.time() - t0
            perm = t.payload.astype(np.uint32)
            name = f"{mode}/{kind}/n{n}/k{k}/s{seed}"
            out[name] = {
                "kind": kind, "n": n, "k": k, "seed": seed, "mode": mode, "input_sha256": sha(pts),
                "perm_sha256": sha(perm), "perm_head": perm[:32].tolist(),
                "coords_sha256": sha(t.coords),
                "split_dims_sha256": sha(t.split_dims.astype(np.uint8)) if mode == "widest" else None,
                "reference_seconds": round(dt, 3), "source": "reference",
            }
            print(name, round(dt, 2), flush=True)
    with open(os.path.join(HERE, "hashes_f64.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
        f.write("\n")


if __name__ == "__main__":
    main()
