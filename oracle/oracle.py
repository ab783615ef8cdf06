"""CPU oracle for the k-d tree build -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker
(or the timed CPU baseline), never as the thing shipped.  The product path
(``paper_2211_00120_b200``) never imports it.

Contents
- ``build_rr`` / ``build_widest``: ctypes front of ``lbkd_oracle.c``, a C
  restatement of the reference's tag-and-sort loop
  (/root/reference/pkg/src/lbkd/builder.py:200-236, widest.py:134-191).
- ``check_valid`` / ``validity_witness``: numpy restatement of
  verify.check_valid (/root/reference/pkg/src/lbkd/verify.py:195-245) and of
  its witness rescan (:226-243).
- ``brute_subtree_boxes``: restatement of verify.brute_subtree_boxes
  (verify.py:347-374).
- ``treemath`` scalar helpers restated from treemath.py:46-140.
- ``brute_knn`` / ``brute_radius``: restatements of verify.brute_knn /
  brute_radius (verify.py:305-320) with the distance accumulation of
  verify._squared_distances (:295-302) -- the checker of the GPU queries.

Parity pin: tests/test_oracle.py checks these against tests/golden/*, which
tests/golden/make_golden.py produced by running the reference itself.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liblbkd_oracle.so")
_lib = None


def build_lib() -> str:
    """Compile lbkd_oracle.c with the committed Makefile (gcc, no GPU)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        srcs = [os.path.join(_HERE, f) for f in ("lbkd_oracle.c", "lbkd_recursive.cpp", "Makefile")]
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
                os.path.getmtime(f) for f in srcs if os.path.exists(f)):
            build_lib()
        lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        lib.oracle_build_rr.argtypes = [p, ctypes.c_int64, ctypes.c_int, p, p, p]
        lib.oracle_build_rr.restype = ctypes.c_int
        lib.oracle_build_widest.argtypes = [p, ctypes.c_int64, ctypes.c_int, p, p]
        lib.oracle_build_widest.restype = ctypes.c_int
        lib.oracle_rec_build_f32.argtypes = [p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, p, p, ctypes.c_int]
        lib.oracle_rec_build_f32.restype = ctypes.c_int
        lib.oracle_rec_build_f64.argtypes = [p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, p, p, ctypes.c_int]
        lib.oracle_rec_build_f64.restype = ctypes.c_int
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_threads.restype = ctypes.c_int
        lib.oracle_set_threads(0)
        _lib = lib
    return _lib


def set_threads(t: int) -> int:
    lib = _load()
    lib.oracle_set_threads(int(t))
    return lib.oracle_threads()


def threads() -> int:
    return _load().oracle_threads()


def _as_points(points) -> np.ndarray:
    pts = np.asarray(points)
    if pts.ndim == 1:
        pts = pts.reshape(-1, 1)
    f = np.ascontiguousarray(pts, dtype=np.float32)
    if pts.dtype != np.float32 and not np.array_equal(f.astype(pts.dtype), pts):
        raise ValueError("oracle works on float32-representable coordinates")
    return f


def build_rr(points, trace: bool = False):
    """Round-robin build. Returns perm (uint32, node -> input row).

    With ``trace=True`` also returns (tags, idx) of shape (phases, n) in the
    BuildRecorder(capture=True) phase order (builder.py:219-235).
    """
    pts = _as_points(points)
    n, k = pts.shape
    perm = np.empty(n, dtype=np.uint32)
    if n == 0:
        return (perm, None, None) if trace else perm
    lib = _load()
    if trace:
        levels = n.bit_length()
        phases = 2 * levels
        tags = np.empty((phases, n), dtype=np.uint32)
        idx = np.empty((phases, n), dtype=np.uint32)
        rc = lib.oracle_build_rr(pts.ctypes.data, n, k, perm.ctypes.data, tags.ctypes.data, idx.ctypes.data)
        assert rc == 0
        return perm, tags, idx
    rc = lib.oracle_build_rr(pts.ctypes.data, n, k, perm.ctypes.data, None, None)
    assert rc == 0
    return perm


def build_widest(points):
    """Widest-dimension build. Returns (perm uint32, split_dims uint8)."""
    pts = _as_points(points)
    n, k = pts.shape
    perm = np.empty(n, dtype=np.uint32)
    dims = np.zeros(n, dtype=np.uint8)
    if n == 0:
        return perm, dims
    rc = _load().oracle_build_widest(pts.ctypes.data, n, k, perm.ctypes.data, dims.ctypes.data)
    assert rc == 0
    return perm, dims


def rec_build(points, widest: bool = False, threads: int = 0):
    """Recursive median-placement oracle (lbkd_recursive.cpp, restating
    verify.reference_build, verify.py:121-168), threaded over subtrees.

    float32 input is used as is; anything else is promoted to float64 like the
    reference's ingest (builder.py:131-133).  Returns perm (uint32), and for
    ``widest`` also split_dims (uint8)."""
    pts = np.asarray(points)
    if pts.ndim == 1:
        pts = pts.reshape(-1, 1)
    n, k = pts.shape
    perm = np.empty(n, dtype=np.uint32)
    dims = np.zeros(n, dtype=np.uint8)
    if n:
        lib = _load()
        if pts.dtype == np.float32:
            pts = np.ascontiguousarray(pts)
            rc = lib.oracle_rec_build_f32(pts.ctypes.data, n, k, int(widest), perm.ctypes.data,
                                          dims.ctypes.data if widest else None, int(threads))
        else:
            pts = np.ascontiguousarray(pts, dtype=np.float64)
            rc = lib.oracle_rec_build_f64(pts.ctypes.data, n, k, int(widest), perm.ctypes.data,
                                          dims.ctypes.data if widest else None, int(threads))
        assert rc == 0, rc
    return (perm, dims) if widest else perm


def timed_build(points, mode: str = "rr") -> float:
    """Wall seconds of one oracle build (the bench CPU baseline)."""
    t0 = time.perf_counter()
    if mode == "rr":
        build_rr(points)
    else:
        build_widest(points)
    return time.perf_counter() - t0


# --- treemath restated (treemath.py:46-140) ---------------------------------

def level(i: int) -> int:
    return (i + 1).bit_length() - 1


def num_levels(n: int) -> int:
    return n.bit_length()


def subtree_size(s: int, n: int) -> int:
    shift = num_levels(n) - level(s) - 1
    width = 1 << shift
    first = ((s + 1) << shift) - 1
    return width - 1 + min(max(0, n - first), width)


def segment_begin(s: int, n: int) -> int:
    lvl = level(s)
    lvls = num_levels(n)
    shift = lvls - lvl - 1
    top = (1 << lvl) - 1
    nls = s - top
    bottom_have = n - ((1 << (lvls - 1)) - 1)
    return top + nls * ((1 << shift) - 1) + min(nls << shift, bottom_have)


# --- verify restated ----------------------------------------------------------

def node_split_dims(n: int, k: int, split_dims=None) -> np.ndarray:
    """verify._node_split_dims (verify.py:186-192)."""
    if split_dims is not None:
        return np.asarray(split_dims).astype(np.int64)
    levels = np.floor(np.log2(np.arange(n, dtype=np.float64) + 1)).astype(np.int64)
    # exact integer levels (log2 float rounding guard)
    idx = np.arange(n, dtype=np.int64) + 1
    levels = np.where((1 << (levels + 1)) <= idx, levels + 1, levels)
    levels = np.where((1 << levels) > idx, levels - 1, levels)
    return levels % k


def check_valid(coords, split_dims=None) -> bool:
    """verify.check_valid (verify.py:195-245): every node against every
    ancestor plane, closed on both sides.  Returns True/False."""
    coords = np.asarray(coords)
    n, k = coords.shape
    if n <= 1:
        return True
    dims = node_split_dims(n, k, split_dims)
    rows = np.arange(n)
    cur = rows.copy()
    for _ in range(num_levels(n) - 1):
        live = cur > 0
        par = np.where(live, (cur - 1) >> 1, 0)
        dp = dims[par]
        own = coords[rows, dp]
        plane = coords[par, dp]
        is_left = (cur & 1) == 1
        bad = np.where(is_left, own > plane, own < plane) & live
        if bad.any():
            return False
        cur = par
    return True


def validity_witness(coords, split_dims=None):
    """The witness of verify.check_valid's deterministic rescan
    (verify.py:226-243): (descendant, ancestor, dim) of the lowest violating
    node and its nearest violated ancestor, or None for a valid tree."""
    coords = np.asarray(coords)
    n, k = coords.shape
    if check_valid(coords, split_dims):
        return None
    dims = node_split_dims(n, k, split_dims)
    for d in range(1, n):
        a = d
        while a > 0:
            p = (a - 1) >> 1
            dp = int(dims[p])
            own, plane = coords[d, dp], coords[p, dp]
            if (a & 1 == 1 and own > plane) or (a & 1 == 0 and own < plane):
                return d, p, dp
            a = p
    return None


def brute_subtree_boxes(coords, split_dims=None):
    """verify.brute_subtree_boxes (verify.py:347-374), float64 boxes."""
    coords = np.asarray(coords, dtype=np.float64)
    n, k = coords.shape
    lo = np.empty((n, k))
    hi = np.empty((n, k))
    if n == 0:
        return lo, hi
    dims = node_split_dims(n, k, split_dims)
    lo[0] = coords.min(axis=0)
    hi[0] = coords.max(axis=0)
    for s in range(n):
        d = dims[s]
        plane = coords[s, d]
        lc = 2 * s + 1
        if lc < n:
            lo[lc] = lo[s]
            hi[lc] = hi[s]
            hi[lc, d] = min(hi[lc, d], plane)
        if lc + 1 < n:
            lo[lc + 1] = lo[s]
            hi[lc + 1] = hi[s]
            lo[lc + 1, d] = max(lo[lc + 1, d], plane)
    return lo, hi


# ---------------------------------------------------------------------------
# query checkers (verify.py:295-320)

def squared_distances(coords, query) -> np.ndarray:
    """verify._squared_distances (verify.py:295-302): float64, accumulated
    dim by dim in the traversal kernels' order."""
    coords = np.asarray(coords, dtype=np.float64)
    query = np.asarray(query, dtype=np.float64).reshape(-1)
    d2 = np.zeros(coords.shape[0], dtype=np.float64)
    for j in range(coords.shape[1]):
        t = query[j] - coords[:, j]
        d2 += t * t
    return d2


def brute_knn(coords, query, m: int):
    """verify.brute_knn (verify.py:305-312): the m nearest rows by full scan
    as (index, dist2) pairs ordered by (dist2, index)."""
    d2 = squared_distances(coords, query)
    order = np.lexsort((np.arange(d2.shape[0]), d2))
    take = min(m, d2.shape[0])
    return [(int(i), float(d2[i])) for i in order[:take]]


def brute_radius(coords, query, radius: float) -> np.ndarray:
    """verify.brute_radius (verify.py:315-320): every index with
    dist2 <= radius**2, ascending int64."""
    d2 = squared_distances(coords, query)
    return np.nonzero(d2 <= float(radius) ** 2)[0].astype(np.int64)
