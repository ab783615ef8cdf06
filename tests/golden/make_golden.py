"""Generate golden vectors by running the reference package itself.

Runs ONLY in the authoring container, where the read-only reference lives at
/root/reference (it does not exist on the GPU box; the outputs below are
committed so nothing at test time needs it).

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py            # small + medium
    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden.py --big      # 10M/100M hashes

Outputs (tests/golden/):
  walkthrough.npz     the §5 walkthrough: input + every BuildRecorder phase
                      (tags, coords) -- reference verify.py:26-91 replayed
                      through builder.build_round_robin(recorder=capture)
  small.npz           ~300 small builds (RR + widest): full perm/split_dims
  hashes.json         sha256 of the reference output permutation (uint32
                      little endian) and split dims for medium/large cases,
                      plus sha256 of the generated input
Each case names its generator (paper_2211_00120_b200.datagen) so tests can
regenerate the exact input.
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
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")
os.environ.setdefault("LBKD_BACKEND", "numba")

import lbkd  # noqa: E402  (the reference)
from lbkd import builder, verify  # noqa: E402

from paper_2211_00120_b200 import datagen  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def ref_build(pts: np.ndarray, mode: str):
    if mode == "rr":
        t = lbkd.build_round_robin(pts, pts.shape[1])
        return t.payload.astype(np.uint32), None
    t = lbkd.build_widest(pts, pts.shape[1])
    return t.payload.astype(np.uint32), t.split_dims.astype(np.uint8)


def walkthrough():
    pts = verify.WALKTHROUGH_POINTS.astype(np.float32)
    rec = builder.BuildRecorder(capture=True)
    tree = lbkd.build_round_robin(pts, 2, recorder=rec)
    tags = np.stack([s.tags for s in rec.snapshots]).astype(np.uint32)
    coords = np.stack([s.coords for s in rec.snapshots]).astype(np.float32)
    events = np.array([s.event for s in rec.snapshots])
    iters = np.array([s.iteration for s in rec.snapshots], dtype=np.int32)
    # cross-check against the hand tables in verify.WALKTHROUGH_STATES
    for snap, (_, t, xs, ys) in zip(rec.snapshots, verify.WALKTHROUGH_STATES):
        assert snap.tags.tolist() == list(t)
        assert snap.coords[:, 0].tolist() == list(map(float, xs))
        assert snap.coords[:, 1].tolist() == list(map(float, ys))
    np.savez(
        os.path.join(HERE, "walkthrough.npz"),
        points=pts,
        tags=tags,
        coords=coords,
        events=events,
        iterations=iters,
        perm=tree.payload.astype(np.uint32),
    )


def small_cases():
    rng = np.random.default_rng(20221101)
    cases = []
    sizes = list(range(1, 40)) + [63, 64, 65, 127, 128, 129, 255, 256, 257, 511, 1000, 1023, 1024, 1025, 4095, 4096, 4097, 8191, 8192, 8193, 12345, 20000]
    kinds = ["uniform", "ties", "signed_zero", "clustered", "int3"]
    for n in sizes:
        for mode in ("rr", "widest"):
            k = int(rng.integers(1, 5))
            kind = kinds[int(rng.integers(0, len(kinds)))]
            seed = int(rng.integers(0, 1 << 30))
            cases.append((kind, n, k, seed, mode))
    # explicit edge cases
    for k in (1, 2, 3, 4, 5, 8):
        cases.append(("uniform", 777, k, 5, "rr"))
        cases.append(("uniform", 777, k, 6, "widest"))
        cases.append(("int3", 300, k, 7, "rr"))
        cases.append(("int3", 300, k, 8, "widest"))
    perms, dims, meta = [], [], []
    for kind, n, k, seed, mode in cases:
        pts = gen(kind, n, k, seed)
        perm, sd = ref_build(pts, mode)
        perms.append(perm)
        dims.append(sd if sd is not None else np.zeros(0, np.uint8))
        meta.append((kind, n, k, seed, mode))
    np.savez_compressed(
        os.path.join(HERE, "small.npz"),
        kind=np.array([m[0] for m in meta]),
        n=np.array([m[1] for m in meta], dtype=np.int64),
        k=np.array([m[2] for m in meta], dtype=np.int64),
        seed=np.array([m[3] for m in meta], dtype=np.int64),
        mode=np.array([m[4] for m in meta]),
        perm=np.concatenate(perms),
        split_dims=np.concatenate(dims),
    )
    print(f"small: {len(cases)} cases")


def gen(kind, n, k, seed):
    if kind == "int3":
        return np.random.default_rng(seed).integers(0, 3, size=(n, k)).astype(np.float32)
    return datagen.make(kind, n, k, seed)


MEDIUM = [
    ("uniform", 1_000_000, 3, 0, "rr"),        # config 1
    ("ties", 100_000, 3, 1, "rr"),
    ("signed_zero", 20_000, 2, 2, "rr"),
    ("clustered", 200_000, 3, 3, "rr"),
    ("uniform", 300_000, 2, 4, "rr"),
    ("uniform", 100_000, 4, 5, "rr"),
    ("uniform", 65_537, 3, 6, "rr"),
    ("uniform", 100_000, 3, 7, "widest"),
    ("clustered", 100_000, 3, 8, "widest"),
    ("ties", 50_000, 4, 9, "widest"),
    ("clustered", 1_000_000, 3, 1, "widest"),
    ("signed_zero", 20_000, 3, 10, "widest"),
]

BIG = [
    ("uniform", 10_000_000, 4, 0, "rr"),       # config 3
    ("uniform", 100_000_000, 3, 0, "rr"),      # headline
    ("clustered", 100_000_000, 3, 1, "widest"),  # config 5
    ("uniform", 100_000_000, 2, 0, "rr"),      # config 2
]


def hash_cases(cases):
    path = os.path.join(HERE, "hashes.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for kind, n, k, seed, mode in cases:
        key = f"{mode}/{kind}/n{n}/k{k}/s{seed}"
        if key in out:
            continue
        pts = gen(kind, n, k, seed)
        t0 = time.perf_counter()
        perm, sd = ref_build(pts, mode)
        el = time.perf_counter() - t0
        out[key] = {
            "kind": kind, "n": n, "k": k, "seed": seed, "mode": mode,
            "input_sha256": sha(pts),
            "perm_sha256": sha(perm),
            "perm_head": perm[:64].tolist(),
            "split_dims_sha256": sha(sd) if sd is not None else None,
            "reference_seconds": round(el, 3),
        }
        print(key, f"{el:.1f}s", flush=True)
        json.dump(out, open(path, "w"), indent=1, sort_keys=True)
        del pts, perm, sd


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    # JIT warmup so timings exclude compilation
    lbkd.build_round_robin(np.random.default_rng(0).random((1000, 3)), 3)
    lbkd.build_widest(np.random.default_rng(0).random((1000, 3)), 3)
    if args.big:
        hash_cases(BIG)
        return
    walkthrough()
    small_cases()
    hash_cases(MEDIUM)


if __name__ == "__main__":
    main()
