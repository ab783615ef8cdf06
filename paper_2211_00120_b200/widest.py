"""Widest-dimension build -- drop-in for ``lbkd.widest``.

Same public names as /root/reference/pkg/src/lbkd/widest.py:33-44.  The
small host helpers (packing, boxes) are plain Python like the reference's;
``build_widest`` (widest.py:134-191) runs on the GPU: world-bounds reduction,
per-node child-dim kernel and the same segmented sort as the round-robin
build, keyed by each node's own split dimension.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _native, treemath
from .builder import (
    MAX_POINTS,
    BuildRecorder,
    KdTree,
    _check_host_buffers,
    _check_out_buffers,
    _check_points_tensor,
    _raise_for,
    _record_trace,
    _stream_ptr,
    _torch,
    ingest,
)

__all__ = [
    "Aabb",
    "PackedTag",
    "dim_bits_for",
    "pack_tag",
    "unpack_tag",
    "world_bounds",
    "widest_dim",
    "subtree_bounds",
    "build_widest",
    "build_widest_cuda",
]


@dataclass
class Aabb:
    lo: np.ndarray
    hi: np.ndarray

    def copy(self) -> "Aabb":
        return Aabb(self.lo.copy(), self.hi.copy())

    def widths(self) -> np.ndarray:
        return self.hi - self.lo


class PackedTag(NamedTuple):
    node: int
    dim: int


def dim_bits_for(k: int) -> int:
    if k < 1:
        raise ValueError("dimension count must be at least 1")
    return (k - 1).bit_length()


def pack_tag(node: int, dim: int, dim_bits: int) -> int:
    if not 0 <= dim < max(1 << dim_bits, 1):
        raise ValueError("split dimension does not fit the reserved bits")
    return (node << dim_bits) | dim


def unpack_tag(value: int, dim_bits: int) -> PackedTag:
    return PackedTag(value >> dim_bits, value & ((1 << dim_bits) - 1))


def world_bounds(coords: np.ndarray) -> Aabb:
    coords = np.asarray(coords)
    if coords.shape[0] < 1:
        raise ValueError("bounding box of zero points is undefined")
    return Aabb(coords.min(axis=0).astype(np.float64), coords.max(axis=0).astype(np.float64))


def widest_dim(box: Aabb) -> int:
    """First maximum of the float64 widths (ties toward the lower index)."""
    return int(np.argmax(box.widths()))


def subtree_bounds(tree_coords, split_dims, node: int, world: Aabb) -> Aabb:
    """Clip the world box by every ancestor plane of ``node``."""
    box = world.copy()
    a = node
    while a > 0:
        p = (a - 1) >> 1
        d = int(split_dims[p])
        plane = tree_coords[p, d]
        if a & 1:
            box.hi[d] = min(box.hi[d], plane)
        else:
            box.lo[d] = max(box.lo[d], plane)
        a = p
    return box


def build_widest_cuda(points, *, out=None, perm=None, split_dims=None, stream=None, check_finite: bool = True,
                      trace=None):
    """Device-resident widest build on a (n, k) float32 or float64 CUDA
    tensor (float64: lbkd_build_widest_f64).

    Returns (out, perm, split_dims)."""
    torch = _torch()
    _check_points_tensor(torch, points)
    _check_out_buffers(torch, points, out, perm, split_dims)
    if trace is not None:
        L = treemath.num_levels(points.shape[0])
        if (trace.device != points.device or trace.dtype != torch.int32 or not trace.is_contiguous()
                or trace.numel() < max(L, 1) * points.shape[0]):
            raise ValueError("trace must be a contiguous int32 tensor of num_levels(n) * n entries")
    n, k = points.shape
    dev = points.device.index if points.device.index is not None else torch.cuda.current_device()
    if out is None:
        out = torch.empty_like(points)
    if perm is None:
        perm = torch.empty(n, dtype=torch.int32, device=points.device)
    if split_dims is None:
        split_dims = torch.zeros(n, dtype=torch.uint8, device=points.device)
    lib = _native.load()
    ctx = _native.context(dev)
    lib.lbkd_set_check(ctx, 1 if check_finite else 0)
    with torch.cuda.device(dev):
        sp = _stream_ptr(torch, stream)
        f64 = points.dtype == torch.float64
        if trace is None:
            fn = lib.lbkd_build_widest_f64 if f64 else lib.lbkd_build_widest
            rc = fn(ctx, points.data_ptr(), out.data_ptr(), n, k, perm.data_ptr(), split_dims.data_ptr(), sp)
        else:
            fn = lib.lbkd_build_widest_f64_trace if f64 else lib.lbkd_build_widest_trace
            rc = fn(ctx, points.data_ptr(), out.data_ptr(), n, k, perm.data_ptr(), split_dims.data_ptr(),
                    trace.data_ptr(), sp)
    _raise_for(rc, "lbkd_build_widest", n, k, widest=True)
    return out, perm, split_dims


def build_widest_host(points, out, perm, split_dims, *, device: int = 0, stream=None) -> None:
    """Pipelined widest build from HOST memory through lbkd_build_widest_host.

    ``points`` / ``out``: (n, k) float32, ``perm``: (n,) int32, ``split_dims``:
    (n,) uint8 CPU tensors, all pinned for overlap.  The call only enqueues
    H2D -> build -> D2H; consecutive calls overlap their copies with the
    neighbouring builds.  The buffers are valid after ``builder.host_join``.
    """
    torch = _torch()
    _check_host_buffers(torch, points, out, perm, split_dims)
    n, k = points.shape
    lib = _native.load()
    ctx = _native.context(device)
    with torch.cuda.device(device):
        rc = lib.lbkd_build_widest_host(ctx, points.data_ptr(), out.data_ptr(), n, k, perm.data_ptr(),
                                        split_dims.data_ptr(), _stream_ptr(torch, stream))
    _raise_for(rc, "lbkd_build_widest_host", n, k, widest=True)


def build_widest(points, k: int | None = None, payload=None, *, skip_prefix: bool = False,
                 recorder: BuildRecorder | None = None) -> KdTree:
    """Drop-in for lbkd.build_widest (widest.py:134-191)."""
    raw = np.asarray(points)
    if raw.ndim in (1, 2):
        n0 = raw.shape[0]
        k0 = raw.shape[1] if raw.ndim == 2 else 1
        # same capacity rule as the reference, checked before any copy
        if n0 > 0 and k0 > 0 and (n0 << dim_bits_for(k0)) > MAX_POINTS:
            raise ValueError(f"{n0} points with {k0} dimensions exceed the 32-bit tag capacity")
    coords, payload = ingest(raw, k, payload)
    n, kd = coords.shape
    dim_dtype = np.min_scalar_type(max(kd - 1, 0))
    if n == 0:
        if recorder is not None:
            recorder.tags_allocated(np.zeros(0, dtype=np.uint32))
        return KdTree(coords.astype(np.float64), payload, np.zeros(0, dtype=dim_dtype))
    torch = _torch()
    capture = recorder is not None and recorder.capture
    dev = torch.cuda.current_device()
    d_pts = torch.from_numpy(coords).to(device=f"cuda:{dev}")
    trace = None
    if capture:
        cap = int(_native.load().lbkd_single_cta_capacity(kd, 1))
        if n > cap:
            raise ValueError(f"BuildRecorder(capture=True) is supported for n <= {cap}")
        trace = torch.zeros(treemath.num_levels(n) * n, dtype=torch.int32, device=d_pts.device)
    out, perm, dims = build_widest_cuda(d_pts, trace=trace)
    out_h = out.cpu().numpy()
    perm_h = perm.cpu().numpy().view(np.uint32).astype(np.int64)
    dims_h = dims.cpu().numpy()
    if recorder is not None:
        if capture:
            db = dim_bits_for(kd)
            tr = trace.cpu().numpy().view(np.uint32).reshape(-1, n)

            def pack(nodes):
                return ((nodes << db) | dims_h[nodes].astype(np.int64)).astype(np.uint32)

            _record_trace(recorder, coords, out_h, perm_h, tr, n, kd, tags_of_node=pack)
        else:
            L = treemath.num_levels(n)
            recorder.tags_allocated(np.zeros(n, dtype=np.uint32))
            recorder.sort_phases += L
            recorder.update_phases += L - 1
    return KdTree(out_h.astype(np.float64), payload[perm_h], dims_h.astype(dim_dtype))
