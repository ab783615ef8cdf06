"""Golden hash of BASELINE config 4: 1B clustered float3, round-robin.

The reference itself needs ~90 GB and hours at this size,
so the expected permutation comes from the threaded recursive oracle
(oracle/lbkd_recursive.cpp, a restatement of verify.reference_build,
/root/reference/pkg/src/lbkd/verify.py:121-168).  That oracle is pinned
first: ``--validate`` re-runs it on every reference-generated case of
hashes.json (1M-100M, ties, +-0.0, clustered negatives, widest) and refuses
to write the 1B entry unless all of them match the reference's own hashes.

    python tests/golden/make_golden_1b.py [--n N] [--validate]

Writes/updates the entry ``rr/clustered/n<N>/k3/s0`` of hashes.json with
``"source": "recursive-oracle"`` (the other entries say "reference").
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import oracle  # noqa: E402
from paper_2211_00120_b200 import datagen  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def validate(hashes) -> dict:
    from golden_util import gen_case

    out = {}
    for name, c in sorted(hashes.items(), key=lambda kv: kv[1]["n"]):
        if c.get("source", "reference") != "reference":
            continue
        pts = gen_case(c)
        assert sha(pts) == c["input_sha256"], name
        t = time.time()
        if c["mode"] == "widest":
            perm, dims = oracle.rec_build(pts, widest=True)
            ok = sha(perm) == c["perm_sha256"] and sha(dims) == c["split_dims_sha256"]
        else:
            ok = sha(oracle.rec_build(pts)) == c["perm_sha256"]
        out[name] = {"ok": bool(ok), "seconds": round(time.time() - t, 2)}
        print(name, out[name], flush=True)
        if not ok:
            raise SystemExit(f"recursive oracle disagrees with the reference on {name}")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000_000)
    ap.add_argument("--validate", action="store_true")
    args = ap.parse_args()
    path = os.path.join(HERE, "hashes.json")
    hashes = json.load(open(path))
    checked = validate(hashes) if args.validate else None
    n, k, seed, kind = args.n, 3, 0, "clustered"
    t = time.time()
    pts = datagen.make(kind, n, k, seed)
    gen_s = time.time() - t
    in_sha = sha(pts)
    t = time.time()
    perm = oracle.rec_build(pts)
    build_s = time.time() - t
    entry = {
        "input_sha256": in_sha, "k": k, "kind": kind, "mode": "rr", "n": n,
        "perm_head": perm[:64].tolist(), "perm_sha256": sha(perm), "seed": seed,
        "split_dims_sha256": None, "source": "recursive-oracle",
        "oracle_seconds": round(build_s, 1), "oracle_threads": os.cpu_count(),
        "generate_seconds": round(gen_s, 1),
        "validated_against": sorted(checked) if checked else None,
    }
    hashes[f"rr/{kind}/n{n}/k{k}/s{seed}"] = entry
    with open(path, "w") as f:
        json.dump(hashes, f, indent=1, sort_keys=True)
        f.write("\n")
    print(json.dumps(entry))


if __name__ == "__main__":
    main()
