"""Whole-tree checks on the GPU -- drop-in for ``lbkd.verify.check_valid`` and
``lbkd.verify.brute_subtree_boxes``.

Mirrors /root/reference/pkg/src/lbkd/verify.py: ``ValidityReport`` (:170-183),
``check_valid(tree)`` (:195-245: same verdict, same witness -- lowest
descendant, then nearest ancestor -- and the same message) and
``brute_subtree_boxes(tree)`` (:347-374).  Both run as CUDA kernels behind the
C-ABI (``lbkd_check_valid`` / ``lbkd_subtree_boxes``, csrc/verify.cu), so a
100M-point tree is validated where it was built; ``check_valid_cuda`` /
``subtree_boxes_cuda`` take the device tensors directly.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .builder import KdTree, _stream_ptr, _torch


@dataclass
class ValidityReport:
    """Outcome of a whole-tree ordering check (verify.py:170-183)."""

    valid: bool
    descendant: int | None = None
    ancestor: int | None = None
    dim: int | None = None
    message: str = ""


def _check(torch, pts, split_dims):
    if (pts.device.type != "cuda" or pts.dtype not in (torch.float32, torch.float64) or pts.dim() != 2
            or not pts.is_contiguous()):
        raise ValueError("tree points must be a contiguous (n, k) float32 or float64 CUDA tensor")
    if split_dims is not None and (split_dims.dtype != torch.uint8 or split_dims.numel() != pts.shape[0]):
        raise ValueError("split_dims must be a uint8 CUDA tensor with one entry per node")


def check_valid_cuda(tree_points, *, split_dims=None, stream=None):
    """(descendant, ancestor, dim) of the first violation, or None if valid."""
    torch = _torch()
    _check(torch, tree_points, split_dims)
    n, k = tree_points.shape
    wit = torch.empty(3, dtype=torch.int64, device=tree_points.device)
    scratch = torch.empty(1, dtype=torch.int64, device=tree_points.device)
    with torch.cuda.device(tree_points.device):
        lib = _native.load()
        fn = lib.lbkd_check_valid_f64 if tree_points.dtype == torch.float64 else lib.lbkd_check_valid
        rc = fn(tree_points.data_ptr() if n else None, n, k,
                                             split_dims.data_ptr() if split_dims is not None else None,
                                             wit.data_ptr(), scratch.data_ptr(), _stream_ptr(torch, stream))
    _native.check(rc, "lbkd_check_valid")
    d, a, dim = (int(v) for v in wit.cpu().tolist())
    return None if d < 0 else (d, a, dim)


def subtree_boxes_cuda(tree_points, *, split_dims=None, stream=None):
    """(lo, hi): float64 (n, k) CUDA tensors of every node's clipped box."""
    torch = _torch()
    _check(torch, tree_points, split_dims)
    n, k = tree_points.shape
    lo = torch.empty((n, k), dtype=torch.float64, device=tree_points.device)
    hi = torch.empty((n, k), dtype=torch.float64, device=tree_points.device)
    with torch.cuda.device(tree_points.device):
        lib = _native.load()
        fn = lib.lbkd_subtree_boxes_f64 if tree_points.dtype == torch.float64 else lib.lbkd_subtree_boxes
        rc = fn(tree_points.data_ptr() if n else None, n, k,
                                               split_dims.data_ptr() if split_dims is not None else None,
                                               lo.data_ptr(), hi.data_ptr(), _stream_ptr(torch, stream))
    _native.check(rc, "lbkd_subtree_boxes")
    return lo, hi


def _device_tree(tree: KdTree):
    from .queries import _device_tree as dev_tree

    return dev_tree(_torch(), tree)


def check_valid(tree: KdTree) -> ValidityReport:
    """Every node against every ancestor's split plane (verify.py:195-245)."""
    if tree.n <= 1:
        return ValidityReport(True)
    pts, dims = _device_tree(tree)
    w = check_valid_cuda(pts, split_dims=dims)
    if w is None:
        return ValidityReport(True)
    d, p, dp = w
    a = d
    while (a - 1) >> 1 != p:  # the child of p on d's path decides the side
        a = (a - 1) >> 1
    own = tree.coords[d, dp]
    plane = tree.coords[p, dp]
    side = "left" if a & 1 == 1 else "right"
    return ValidityReport(
        False, descendant=d, ancestor=p, dim=dp,
        message=(f"node {d} ({own!r}) is in the {side} subtree of node"
                 f" {p} but crosses its dim-{dp} plane ({plane!r})"),
    )


def brute_subtree_boxes(tree: KdTree) -> tuple[np.ndarray, np.ndarray]:
    """Bounding boxes of every node's subtree, clipped top-down
    (verify.py:347-374): (lo, hi) float64 arrays of shape (n, k)."""
    n, k = tree.coords.shape
    if n == 0:
        return np.empty((0, k), np.float64), np.empty((0, k), np.float64)
    pts, dims = _device_tree(tree)
    lo, hi = subtree_boxes_cuda(pts, split_dims=dims)
    return lo.cpu().numpy(), hi.cpu().numpy()


__all__ = ["ValidityReport", "check_valid", "check_valid_cuda", "brute_subtree_boxes", "subtree_boxes_cuda"]
