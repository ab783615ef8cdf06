"""Device timing of batched kNN / radius queries (development aid)."""
import sys
import numpy as np
import torch
sys.path.insert(0, __file__.rsplit('/tools/', 1)[0])
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import datagen, queries


def timed(f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return min(ts)


RESULTS = []


def run(n, nq, k=3, kind="uniform", sort_queries=False):
    pts = datagen.make(kind, n, k, seed=0)
    out, perm = kd.build_round_robin_cuda(torch.from_numpy(pts).cuda())
    qn = np.random.default_rng(1).random((nq, k))
    if sort_queries:  # spatially coherent batch: sort by a coarse grid cell
        cell = np.floor(qn * 64).astype(np.int64)
        key = (cell[:, 0] * 64 + cell[:, 1]) * 64 + cell[:, 2]
        qn = qn[np.argsort(key, kind="stable")]
    q = torch.from_numpy(np.ascontiguousarray(qn)).cuda()
    tag = f"n={n} nq={nq} k={k} {kind}{' sorted' if sort_queries else ''}"
    for m in (1, 8, 32, 64):
        ms = timed(lambda: queries.knn_cuda(out, q, m))
        print(f"knn  m={m:3d} {tag}: {ms:8.3f} ms  {nq / ms / 1e3:8.2f} Mq/s", flush=True)
        RESULTS.append({"query": "knn", "m": m, "tree_n": n, "nq": nq, "k": k, "kind": kind,
                        "coherent": sort_queries, "ms": ms, "mq_per_s": nq / ms / 1e3})
    r = (8 / n / (4 / 3 * np.pi)) ** (1 / 3)  # ~8 expected hits
    ms = timed(lambda: queries.radius_cuda(out, q, r))
    print(f"radius ~8 hits {tag}: {ms:8.3f} ms  {nq / ms / 1e3:8.2f} Mq/s", flush=True)
    RESULTS.append({"query": "radius", "radius": r, "tree_n": n, "nq": nq, "k": k, "kind": kind,
                    "coherent": sort_queries, "ms": ms, "mq_per_s": nq / ms / 1e3})


if __name__ == "__main__":
    import json
    run(1_000_000, 1_000_000)
    run(10_000_000, 1_000_000)
    run(10_000_000, 1_000_000, sort_queries=True)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as fh:
            json.dump({"device": torch.cuda.get_device_name(), "timing": "CUDA events, min of 5 after warm-up",
                       "queries": "uniform [0,1)^k float64, one thread per query", "results": RESULTS}, fh, indent=1)
