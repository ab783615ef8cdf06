"""Helpers to regenerate the inputs of the committed golden cases."""

from __future__ import annotations

import os

import numpy as np

from paper_2211_00120_b200 import datagen

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gen_case(case) -> np.ndarray:
    kind, n, k, seed = case["kind"], int(case["n"]), int(case["k"]), int(case["seed"])
    if kind == "int3":
        return np.random.default_rng(seed).integers(0, 3, size=(n, k)).astype(np.float32)
    return datagen.make(kind, n, k, seed)


def small_cases():
    g = np.load(os.path.join(GOLDEN, "small.npz"))
    off = 0
    out = []
    doff = 0
    for i in range(len(g["n"])):
        n = int(g["n"][i])
        mode = str(g["mode"][i])
        case = {
            "kind": str(g["kind"][i]), "n": n, "k": int(g["k"][i]),
            "seed": int(g["seed"][i]), "mode": mode,
            "perm": g["perm"][off:off + n],
            "name": f"{mode}-{g['kind'][i]}-n{n}-k{int(g['k'][i])}-s{int(g['seed'][i])}",
        }
        off += n
        if mode == "widest":
            case["split_dims"] = g["split_dims"][doff:doff + n]
            doff += n
        out.append(case)
    return out
