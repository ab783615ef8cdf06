"""A kernel module for the reference's plugin seam, on the B200.

The reference dispatches its per-level update kernels and its query
traversals through ``lbkd.accel.get_kernels()``
(/root/reference/pkg/src/lbkd/accel.py:48-58), which returns a module with
four functions (kernels_numpy.py:41-245, kernels_numba.py:21-110).  This
module has the same four, with the same signatures and in-place semantics,
backed by the C ABI:

    update_tags_round_robin(tags, n, levels, l)          -> lbkd_update_tags_rr
    update_tags_widest(tags, coords, split_dims, world_lo, world_hi,
                       n, levels, l, dim_bits)            -> lbkd_update_tags_widest
    knn_search(coords, split_dims, k, query, m, out_idx, out_d2) -> lbkd_knn_f64
    radius_search(coords, split_dims, k, query, r2, out_idx)     -> lbkd_radius_*_f64

A maintainer registers it as a third backend (seam 2); the
reference keeps its own sort and loop.  Each call copies its arrays to the
device and the results back -- this seam exists for compatibility, the
whole-build drop-in (``build_round_robin``) is the fast path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("kernels_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _stream(torch):
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def update_tags_round_robin(tags: np.ndarray, n: int, levels: int, l: int) -> None:
    """kernels_numba.update_tags_round_robin (kernels_numba.py:21-46): tags of
    [F(l), n) -> child tags, in place."""
    torch = _torch()
    t = torch.from_numpy(np.ascontiguousarray(tags).view(np.int32)).cuda()
    _native.check(_native.load().lbkd_update_tags_rr(t.data_ptr(), int(n), int(levels), int(l), _stream(torch)),
                  "lbkd_update_tags_rr")
    tags[:] = t.cpu().numpy().view(tags.dtype)


def update_tags_widest(tags, coords, split_dims, world_lo, world_hi, n, levels, l, dim_bits) -> None:
    """kernels_numba.update_tags_widest (kernels_numba.py:49-110): packed child
    tags in place; the pivot of every level-l node writes split_dims[node]."""
    torch = _torch()
    dev = "cuda"
    t = torch.from_numpy(np.ascontiguousarray(tags).view(np.int32)).to(dev)
    c = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.float64)).to(dev)
    sd = torch.from_numpy(np.ascontiguousarray(split_dims).astype(np.uint8)).to(dev)
    lo = torch.from_numpy(np.ascontiguousarray(world_lo, dtype=np.float64)).to(dev)
    hi = torch.from_numpy(np.ascontiguousarray(world_hi, dtype=np.float64)).to(dev)
    k = c.shape[1] if c.dim() == 2 else 1
    rc = _native.load().lbkd_update_tags_widest(t.data_ptr(), c.data_ptr(), int(k), sd.data_ptr(), lo.data_ptr(),
                                                hi.data_ptr(), int(n), int(levels), int(l), int(dim_bits),
                                                _stream(torch))
    _native.check(rc, "lbkd_update_tags_widest")
    tags[:] = t.cpu().numpy().view(tags.dtype)
    split_dims[:] = sd.cpu().numpy().astype(split_dims.dtype)


def _tree(torch, coords, split_dims):
    c = torch.from_numpy(np.ascontiguousarray(coords, dtype=np.float64)).cuda()
    sd = None
    if split_dims is not None and np.asarray(split_dims).shape[0] != 0:
        sd = torch.from_numpy(np.ascontiguousarray(split_dims).astype(np.uint8)).cuda()
    return c, sd


def knn_search(coords, split_dims, k, query, m, out_idx, out_d2) -> int:
    """kernels_numpy.knn_search (kernels_numpy.py:114-195): the min(m, n)
    nearest nodes by (squared distance, node index) into out_idx / out_d2;
    returns how many."""
    torch = _torch()
    n = coords.shape[0]
    if n == 0 or m < 1:
        return 0
    c, sd = _tree(torch, coords, split_dims)
    want = min(int(m), n)
    q = torch.from_numpy(np.ascontiguousarray(query, dtype=np.float64).reshape(1, -1)).cuda()
    idx = torch.empty((1, want), dtype=torch.int64, device="cuda")
    d2 = torch.empty((1, want), dtype=torch.float64, device="cuda")
    rc = _native.load().lbkd_knn_f64(c.data_ptr(), n, int(k), sd.data_ptr() if sd is not None else None,
                                     q.data_ptr(), 1, want, idx.data_ptr(), d2.data_ptr(), _stream(torch))
    _native.check(rc, "lbkd_knn_f64")
    out_idx[:want] = idx.cpu().numpy()[0]
    out_d2[:want] = d2.cpu().numpy()[0]
    return want


def radius_search(coords, split_dims, k, query, r2, out_idx) -> int:
    """kernels_numpy.radius_search (kernels_numpy.py:198-245): every node with
    squared distance <= r2 into out_idx (ascending here; the caller sorts,
    queries.py:77); returns the count."""
    torch = _torch()
    n = coords.shape[0]
    if n == 0:
        return 0
    c, sd = _tree(torch, coords, split_dims)
    lib = _native.load()
    q = torch.from_numpy(np.ascontiguousarray(query, dtype=np.float64).reshape(1, -1)).cuda()
    counts = torch.empty(1, dtype=torch.int64, device="cuda")
    offsets = torch.empty(2, dtype=torch.int64, device="cuda")
    scratch = torch.empty(int(lib.lbkd_radius_scratch_len(1)), dtype=torch.int64, device="cuda")
    dp = sd.data_ptr() if sd is not None else None
    _native.check(lib.lbkd_radius_count_f64(c.data_ptr(), n, int(k), dp, q.data_ptr(), 1, float(r2),
                                            counts.data_ptr(), offsets.data_ptr(), scratch.data_ptr(),
                                            _stream(torch)), "lbkd_radius_count_f64")
    total = int(offsets[1].cpu())
    idx = torch.empty(max(total, 1), dtype=torch.int64, device="cuda")
    _native.check(lib.lbkd_radius_fill_f64(c.data_ptr(), n, int(k), dp, q.data_ptr(), 1, float(r2),
                                           offsets.data_ptr(), idx.data_ptr(), _stream(torch)),
                  "lbkd_radius_fill_f64")
    out_idx[:total] = idx.cpu().numpy()[:total]
    return total
