"""Nearest-neighbour and radius queries -- drop-in for ``lbkd.queries``.

Mirrors /root/reference/pkg/src/lbkd/queries.py: ``Neighbor`` (:21-23),
``knn(tree, query, m)`` (:41-62) and ``radius_query(tree, query, radius)``
(:65-77), same results (ordered by (squared distance, node index); radius hits
ascending, boundary included) and the same ValueError contract.  The
traversal runs on the GPU through the C-ABI (``lbkd_knn`` /
``lbkd_radius_count`` / ``lbkd_radius_fill``, csrc/query.cu), which answers a
whole batch of queries per launch; there is no CPU path.

Three layers:
- ``knn`` / ``radius_query``: the reference's one-query host API.
- ``knn_batch`` / ``radius_batch``: many host queries against one tree.
- ``knn_cuda`` / ``radius_cuda``: device tensors in and out -- e.g. straight
  on the ``out`` tensor of ``build_round_robin_cuda``.
"""

from __future__ import annotations

from typing import NamedTuple

import numpy as np

from . import _native
from .builder import KdTree, _stream_ptr, _torch


class Neighbor(NamedTuple):
    index: int
    dist2: float


def _device_tree(torch, tree: KdTree):
    """float32 level-order rows (+ split dims) of ``tree`` on the current
    device.  The device copy is cached on the tree object together with a
    host snapshot of the arrays it was made from; every call compares the
    tree's current contents with the snapshot (a memory compare, far cheaper
    than the upload), so in-place edits of ``coords`` / ``split_dims`` are
    always seen."""
    dev = torch.cuda.current_device()
    cached = getattr(tree, "_lbkd_device", None)
    if cached is not None:
        cdev, c_coords, c_dims, pts, dims = cached
        same_dims = (c_dims is None and tree.split_dims is None) or (
            c_dims is not None and tree.split_dims is not None and np.array_equal(c_dims, tree.split_dims))
        if cdev == dev and same_dims and np.shape(tree.coords) == c_coords.shape and np.array_equal(
                tree.coords, c_coords):
            return pts, dims
    c64 = np.ascontiguousarray(tree.coords, dtype=np.float64)
    with np.errstate(over="ignore"):
        c32 = c64.astype(np.float32)
    # float32 rows when they are exact (half the bytes), else the float64 rows
    # (trees built from float64 input); the kernels widen to float64 either way
    rows = c32 if np.array_equal(c32, c64) else c64
    pts = torch.from_numpy(rows).to(f"cuda:{dev}")
    dims = None
    snap_dims = None
    if tree.split_dims is not None:
        snap_dims = np.array(tree.split_dims, copy=True)
        dims = torch.from_numpy(np.ascontiguousarray(tree.split_dims, dtype=np.uint8)).to(f"cuda:{dev}")
    tree._lbkd_device = (dev, c64.copy(), snap_dims, pts, dims)
    return pts, dims


def _prep_queries(tree_k: int, queries) -> np.ndarray:
    q = np.asarray(queries, dtype=np.float64)
    if q.ndim == 1:
        q = q.reshape(1, -1)
    if q.ndim != 2 or q.shape[1] != tree_k:
        raise ValueError(f"query has {q.shape[-1] if q.ndim else 1} dimensions, tree has {tree_k}")
    if not np.all(np.isfinite(q)):
        raise ValueError("query coordinates must be finite")
    return np.ascontiguousarray(q)


def _check_tree_tensor(torch, pts, split_dims):
    if (pts.device.type != "cuda" or pts.dtype not in (torch.float32, torch.float64) or pts.dim() != 2
            or not pts.is_contiguous()):
        raise ValueError("tree points must be a contiguous (n, k) float32 or float64 CUDA tensor")
    if split_dims is not None:
        if split_dims.dtype != torch.uint8 or split_dims.numel() != pts.shape[0] or not split_dims.is_contiguous():
            raise ValueError("split_dims must be a contiguous uint8 CUDA tensor with one entry per node")


def knn_cuda(tree_points, queries, m: int, *, split_dims=None, stream=None):
    """Batched kNN on device tensors.

    ``tree_points``: (n, k) float32 or float64 level-order rows; ``split_dims``: uint8
    (n,) for widest trees, None for round-robin; ``queries``: (nq, k) float64.
    Returns (idx int64 (nq, m'), dist2 float64 (nq, m')) with m' = min(m, n),
    each row ordered by (dist2, node index).
    """
    torch = _torch()
    _check_tree_tensor(torch, tree_points, split_dims)
    n, k = tree_points.shape
    if n == 0:
        raise ValueError("nearest-neighbor query on an empty tree")
    if m < 1:
        raise ValueError("neighbor count must be at least 1")
    if queries.dtype != torch.float64 or queries.dim() != 2 or queries.shape[1] != k or not queries.is_contiguous():
        raise ValueError(f"queries must be a contiguous (nq, {k}) float64 CUDA tensor")
    want = min(m, n)
    nq = queries.shape[0]
    idx = torch.empty((nq, want), dtype=torch.int64, device=tree_points.device)
    d2 = torch.empty((nq, want), dtype=torch.float64, device=tree_points.device)
    lib = _native.load()
    with torch.cuda.device(tree_points.device):
        fn = lib.lbkd_knn_f64 if tree_points.dtype == torch.float64 else lib.lbkd_knn
        rc = fn(tree_points.data_ptr(), n, k, split_dims.data_ptr() if split_dims is not None else None,
                queries.data_ptr(), nq, want, idx.data_ptr(), d2.data_ptr(), _stream_ptr(torch, stream))
    _native.check(rc, "lbkd_knn")
    return idx, d2


def radius_cuda(tree_points, queries, radius: float, *, split_dims=None, stream=None):
    """Batched radius search on device tensors.

    Returns (offsets int64 (nq + 1,), idx int64 (total,)): the hits of query
    q, ascending, are ``idx[offsets[q]:offsets[q + 1]]``.  Reads the total
    back to size ``idx`` (one device sync).
    """
    torch = _torch()
    if radius < 0:
        raise ValueError("radius must be non-negative")
    _check_tree_tensor(torch, tree_points, split_dims)
    n, k = tree_points.shape
    if queries.dtype != torch.float64 or queries.dim() != 2 or queries.shape[1] != k or not queries.is_contiguous():
        raise ValueError(f"queries must be a contiguous (nq, {k}) float64 CUDA tensor")
    r2 = float(radius) ** 2  # as queries.py:75
    nq = queries.shape[0]
    dev = tree_points.device
    lib = _native.load()
    counts = torch.empty(max(nq, 1), dtype=torch.int64, device=dev)
    offsets = torch.empty(nq + 1, dtype=torch.int64, device=dev)
    scratch = torch.empty(int(lib.lbkd_radius_scratch_len(nq)), dtype=torch.int64, device=dev)
    dp = split_dims.data_ptr() if split_dims is not None else None
    tp = tree_points.data_ptr() if n else None
    f64 = tree_points.dtype == torch.float64
    count_fn = lib.lbkd_radius_count_f64 if f64 else lib.lbkd_radius_count
    fill_fn = lib.lbkd_radius_fill_f64 if f64 else lib.lbkd_radius_fill
    with torch.cuda.device(dev):
        sp = _stream_ptr(torch, stream)
        _native.check(count_fn(tp, n, k, dp, queries.data_ptr() if nq else None, nq, r2,
                                            counts.data_ptr(), offsets.data_ptr(), scratch.data_ptr(), sp),
                      "lbkd_radius_count")
        (stream if stream is not None else torch.cuda.current_stream()).synchronize()
        total = int(offsets[nq].cpu())
        idx = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
        _native.check(fill_fn(tp, n, k, dp, queries.data_ptr() if nq else None, nq, r2,
                                           offsets.data_ptr(), idx.data_ptr(), sp), "lbkd_radius_fill")
    return offsets, idx[:total]


def knn_batch(tree: KdTree, queries, m: int):
    """kNN for many host queries: (idx int64 (nq, m'), dist2 float64 (nq, m'))."""
    if tree.n == 0:
        raise ValueError("nearest-neighbor query on an empty tree")
    if m < 1:
        raise ValueError("neighbor count must be at least 1")
    q = _prep_queries(tree.k, queries)
    torch = _torch()
    pts, dims = _device_tree(torch, tree)
    idx, d2 = knn_cuda(pts, torch.from_numpy(q).to(pts.device), m, split_dims=dims)
    return idx.cpu().numpy(), d2.cpu().numpy()


def radius_batch(tree: KdTree, queries, radius: float):
    """Radius search for many host queries: (offsets (nq + 1,), idx) int64."""
    if radius < 0:
        raise ValueError("radius must be non-negative")
    q = _prep_queries(tree.k, queries)
    if tree.n == 0:
        return np.zeros(q.shape[0] + 1, dtype=np.int64), np.empty(0, dtype=np.int64)
    torch = _torch()
    pts, dims = _device_tree(torch, tree)
    off, idx = radius_cuda(pts, torch.from_numpy(q).to(pts.device), radius, split_dims=dims)
    return off.cpu().numpy(), idx.cpu().numpy()


def knn(tree: KdTree, query, m: int) -> list[Neighbor]:
    """The ``m`` nearest tree points to ``query``, nearest first
    (queries.py:41-62): ``min(m, n)`` neighbors ordered by (squared distance,
    node index).  Raises on an empty tree."""
    if tree.n == 0:
        raise ValueError("nearest-neighbor query on an empty tree")
    if m < 1:
        raise ValueError("neighbor count must be at least 1")
    q = np.asarray(query, dtype=np.float64).reshape(-1)
    if q.shape[0] != tree.k:
        raise ValueError(f"query has {q.shape[0]} dimensions, tree has {tree.k}")
    idx, d2 = knn_batch(tree, q.reshape(1, -1), m)
    return [Neighbor(int(i), float(d)) for i, d in zip(idx[0], d2[0])]


def radius_query(tree: KdTree, query, radius: float) -> np.ndarray:
    """Indices of all tree points within ``radius`` of ``query``
    (queries.py:65-77): squared distance <= radius**2, int64, ascending;
    an empty tree yields an empty result."""
    if radius < 0:
        raise ValueError("radius must be non-negative")
    if tree.n == 0:
        return np.empty(0, dtype=np.int64)
    q = np.asarray(query, dtype=np.float64).reshape(-1)
    if q.shape[0] != tree.k:
        raise ValueError(f"query has {q.shape[0]} dimensions, tree has {tree.k}")
    _, idx = radius_batch(tree, q.reshape(1, -1), radius)
    return idx


__all__ = ["Neighbor", "knn", "radius_query", "knn_batch", "radius_batch", "knn_cuda", "radius_cuda"]
