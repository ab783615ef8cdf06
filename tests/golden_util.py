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


def query_cases():
    """The reference's answers in golden/queries.npz (make_golden_queries.py),
    one dict per tree: generator parameters, reference payload, queries and
    per query the knn answers for every m in ``ms`` and the radius hits for
    every radius in ``radii``."""
    g = np.load(os.path.join(GOLDEN, "queries.npz"))
    ms = [int(m) for m in g["ms"]]
    nq = int(g["nq"])
    out = []
    po = qo = ko = kc = ro = rc = 0
    for i in range(len(g["n"])):
        n, k = int(g["n"][i]), int(g["k"][i])
        case = {"kind": str(g["kind"][i]), "n": n, "k": k, "seed": int(g["seed"][i]), "mode": str(g["mode"][i])}
        case["name"] = f"{case['mode']}-{case['kind']}-n{n}-k{k}-s{case['seed']}"
        case["payload"] = g["payload"][po:po + n]
        po += n
        case["queries"] = g["queries"][qo:qo + nq * k].reshape(nq, k)
        qo += nq * k
        case["radii"] = [float(r) for r in g["radii"][i]]
        knn, rad = [], []
        for _ in range(nq):
            per_m = {}
            for m in ms:
                c = int(g["knn_cnt"][kc])
                kc += 1
                per_m[m] = [(int(a), float(b)) for a, b in zip(g["knn_idx"][ko:ko + c], g["knn_d2"][ko:ko + c])]
                ko += c
            knn.append(per_m)
            per_r = []
            for _r in case["radii"]:
                c = int(g["rad_cnt"][rc])
                rc += 1
                per_r.append(g["rad_idx"][ro:ro + c])
                ro += c
            rad.append(per_r)
        case["knn"], case["radius"] = knn, rad
        out.append(case)
    return out


# --- float64 inputs (the reference's own dtype; make_golden_f64.py) ---------

def gen_f64(kind: str, n: int, k: int, seed: int) -> np.ndarray:
    """float64 point sets that are NOT float32-representable (so the drop-in
    takes its float64 device path); the reference's CLI bench draws exactly
    ``default_rng(seed).random((n, k))`` (cli.py:176-177)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform64":  # the reference bench's distribution
        return rng.random((n, k))
    if kind == "ties64":  # multiples of 1/1000: duplicates, none float32-exact
        return np.floor(rng.random((n, k)) * 1000) / 1000
    if kind == "signed_zero64":
        vals = np.array([0.0, -0.0, 0.1, -0.1, 0.3])
        return vals[rng.integers(0, len(vals), size=(n, k))]
    if kind == "clustered64":
        cen = rng.random((256, k))
        return cen[rng.integers(0, 256, size=n)] + rng.normal(0.0, 0.01, size=(n, k))
    if kind == "near64":  # distinct values closer than a float32 ulp
        return 1.0 + rng.integers(0, 1 << 12, size=(n, k)) * 2.0 ** -40
    if kind == "range64":  # far outside the float32 range, both signs
        return 10.0 ** rng.uniform(-300, 300, size=(n, k)) * np.where(rng.random((n, k)) < 0.5, -1.0, 1.0)
    if kind == "mixed64":  # one float32-exact dim next to float64 dims
        p = rng.random((n, k))
        p[:, 0] = np.float32(rng.random(n, dtype=np.float32))
        return p
    raise ValueError(kind)


def f64_cases():
    import json

    with open(os.path.join(GOLDEN, "hashes_f64.json")) as f:
        return list(json.load(f).values())
