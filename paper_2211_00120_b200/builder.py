"""Round-robin build entry point -- drop-in for ``lbkd.builder``.

Mirrors the reference interface /root/reference/pkg/src/lbkd/builder.py:
``KdTree`` (:26-60), ``PhaseSnapshot`` (:63-70), ``BuildRecorder`` (:73-105),
``ingest`` (:108-142, same ValueError contract) and ``build_round_robin``
(:200-236, same signature and result).  The build itself runs on the GPU
through the C-ABI library (``_native``); there is no CPU path.

Two layers:
- ``build_round_robin(points, k, payload, *, skip_prefix, recorder)``: the
  reference's host-array API (copies in, builds on the device, copies out).
- ``build_round_robin_cuda(points_tensor, ...)``: device-resident API on
  torch CUDA tensors, no host traffic (what the benchmark's ``value`` times).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native, treemath

MAX_POINTS = treemath.MAX_NODES
MAX_K = 16


@dataclass
class KdTree:
    """Level-order k-d tree: node s at row s, children at 2s+1, 2s+2."""

    coords: np.ndarray
    payload: np.ndarray
    split_dims: np.ndarray | None = None

    @property
    def n(self) -> int:
        return self.coords.shape[0]

    @property
    def k(self) -> int:
        return self.coords.shape[1]

    @property
    def levels(self) -> int:
        return treemath.num_levels(self.n) if self.n else 0

    def split_dim_of(self, s: int) -> int:
        if not 0 <= s < self.n:
            raise ValueError("node index out of range")
        if self.split_dims is not None:
            return int(self.split_dims[s])
        return treemath.level(s) % self.k


@dataclass
class PhaseSnapshot:
    event: str
    iteration: int
    tags: np.ndarray
    coords: np.ndarray


@dataclass
class BuildRecorder:
    """Phase counts and tag storage of a build (builder.py:73-105).

    ``capture=True`` also records (tags, coords) after every phase, rebuilt
    from the device trace; supported for single-CTA builds
    (n <= lbkd_single_cta_capacity), i.e. the small inputs it is meant for.
    """

    capture: bool = False
    sort_phases: int = 0
    update_phases: int = 0
    tag_entries: int = 0
    tag_itemsize: int = 0
    snapshots: list = field(default_factory=list)

    @property
    def tag_bytes(self) -> int:
        return self.tag_entries * self.tag_itemsize

    def tags_allocated(self, tags: np.ndarray) -> None:
        self.tag_entries = tags.shape[0]
        self.tag_itemsize = tags.dtype.itemsize

    def phase(self, event: str, iteration: int, tags: np.ndarray, coords: np.ndarray) -> None:
        if event == "sort":
            self.sort_phases += 1
        elif event == "update":
            self.update_phases += 1
        if self.capture:
            self.snapshots.append(PhaseSnapshot(event, iteration, tags.copy(), coords.copy()))


def ingest(points, k: int | None = None, payload=None):
    """Validate like the reference (builder.py:108-142); return C-contiguous
    (n, k) coordinates and an int64 payload.

    The reference promotes every input to float64.  Inputs that are exactly
    float32-representable (float32 data, small integers, ...) come back as
    float32 -- the fast device path, whose results are identical because the
    promotion is exact; anything else comes back as float64 and is built by
    the float64 device path (lbkd_build_*_f64: per-dimension ranks)."""
    raw = np.asarray(points)
    if raw.ndim not in (1, 2):
        raise ValueError(f"points must be a 2-d array, got shape {raw.shape}")
    n = raw.shape[0]
    if n > MAX_POINTS:
        raise ValueError(f"{n} points exceed the 32-bit tag capacity ({MAX_POINTS})")
    if raw.ndim == 1:
        raw = raw.reshape(-1, 1)
    if k is not None and raw.shape[1] != k:
        raise ValueError(f"expected {k} dimensions, input has {raw.shape[1]}")
    if n > 0 and raw.shape[1] < 1:
        raise ValueError("points must have at least one dimension")
    if raw.shape[1] > MAX_K:
        raise ValueError(f"at most {MAX_K} dimensions are supported")
    if raw.dtype == np.float32:
        coords = np.ascontiguousarray(raw)
    else:
        wide = np.ascontiguousarray(raw, dtype=np.float64)
        if not np.all(np.isfinite(wide)):
            raise ValueError("coordinates must be finite (no NaN or infinity)")
        with np.errstate(over="ignore"):
            narrow = wide.astype(np.float32)
        # -0.0 and +0.0 compare equal here and are both exact in float32
        coords = narrow if np.array_equal(narrow, wide) else wide
    if not np.all(np.isfinite(coords)):
        raise ValueError("coordinates must be finite (no NaN or infinity)")
    if payload is None:
        payload = np.arange(n, dtype=np.int64)
    else:
        payload = np.asarray(payload, dtype=np.int64).copy()
        if payload.shape != (n,):
            raise ValueError("payload must be one integer per point")
    return coords, payload


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the B200 k-d tree builder needs a CUDA device (no CPU fallback)")
    return torch


def _stream_ptr(torch, stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check_points_tensor(torch, points):
    if points.device.type != "cuda" or points.dtype not in (torch.float32, torch.float64) or points.dim() != 2:
        raise ValueError("points must be a 2-d float32 or float64 CUDA tensor")
    if not points.is_contiguous():
        raise ValueError("points must be C-contiguous (n, k)")


def _check_out_buffers(torch, points, out=None, perm=None, split_dims=None):
    """Caller-supplied outputs must match the points exactly: the C ABI takes
    raw pointers and writes n rows / entries into each of them."""
    n, k = points.shape
    if out is not None and (out.device != points.device or out.dtype != points.dtype
                            or tuple(out.shape) != (n, k) or not out.is_contiguous()):
        raise ValueError(f"out must be a contiguous ({n}, {k}) {points.dtype} tensor on {points.device}")
    if perm is not None and (perm.device != points.device or perm.dtype not in (torch.int32, torch.uint32)
                             or tuple(perm.shape) != (n,) or not perm.is_contiguous()):
        raise ValueError(f"perm must be a contiguous ({n},) int32 tensor on {points.device}")
    if split_dims is not None and (split_dims.device != points.device or split_dims.dtype != torch.uint8
                                   or tuple(split_dims.shape) != (n,) or not split_dims.is_contiguous()):
        raise ValueError(f"split_dims must be a contiguous ({n},) uint8 tensor on {points.device}")


def _check_host_buffers(torch, points, out, perm, split_dims=None):
    """Host-pipeline buffers: contiguous CPU tensors of the right dtype and
    shape (the native side copies n rows into / out of each)."""
    for t in (points, out, perm) + ((split_dims,) if split_dims is not None else ()):
        if t.device.type != "cpu" or not t.is_contiguous():
            raise ValueError("host buffers must be contiguous CPU tensors")
    if points.dtype != torch.float32 or points.dim() != 2:
        raise ValueError("points must be a 2-d float32 CPU tensor")
    n, k = points.shape
    if out.dtype != torch.float32 or tuple(out.shape) != (n, k):
        raise ValueError(f"out must be a ({n}, {k}) float32 CPU tensor")
    if perm.dtype not in (torch.int32, torch.uint32) or tuple(perm.shape) != (n,):
        raise ValueError(f"perm must be a ({n},) int32 CPU tensor")
    if split_dims is not None and (split_dims.dtype != torch.uint8 or tuple(split_dims.shape) != (n,)):
        raise ValueError(f"split_dims must be a ({n},) uint8 CPU tensor")


def build_round_robin_cuda(points, *, out=None, perm=None, stream=None, check_finite: bool = True,
                           trace=None):
    """Device-resident build. ``points``: (n, k) float32 or float64 CUDA
    tensor (float64: lbkd_build_rr_f64, the reference's own dtype).

    Returns (out, perm): level-order points (n, k) of the input dtype and the
    input row of each node (uint32 stored in an int32 tensor).  ``out`` may be
    ``points`` itself (in-place reordering).
    """
    torch = _torch()
    _check_points_tensor(torch, points)
    _check_out_buffers(torch, points, out, perm)
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
    lib = _native.load()
    ctx = _native.context(dev)
    lib.lbkd_set_check(ctx, 1 if check_finite else 0)
    with torch.cuda.device(dev):
        sp = _stream_ptr(torch, stream)
        f64 = points.dtype == torch.float64
        if trace is None:
            fn = lib.lbkd_build_rr_f64 if f64 else lib.lbkd_build_rr
            rc = fn(ctx, points.data_ptr(), out.data_ptr(), n, k, perm.data_ptr(), sp)
        else:
            fn = lib.lbkd_build_rr_f64_trace if f64 else lib.lbkd_build_rr_trace
            rc = fn(ctx, points.data_ptr(), out.data_ptr(), n, k, perm.data_ptr(), trace.data_ptr(), sp)
    _raise_for(rc, "lbkd_build_rr", n, k)
    return out, perm


def build_round_robin_host(points, out, perm, *, device: int = 0, stream=None) -> None:
    """Pipelined build from HOST memory through lbkd_build_rr_host.

    ``points`` / ``out``: (n, k) float32 CPU tensors, ``perm``: (n,) int32 CPU
    tensor, all pinned for overlap.  The call only enqueues H2D -> build ->
    D2H; consecutive calls overlap their copies with the previous build.  The
    buffers are valid after :func:`host_join`.
    """
    torch = _torch()
    _check_host_buffers(torch, points, out, perm)
    n, k = points.shape
    lib = _native.load()
    ctx = _native.context(device)
    with torch.cuda.device(device):
        rc = lib.lbkd_build_rr_host(ctx, points.data_ptr(), out.data_ptr(), n, k, perm.data_ptr(),
                                    _stream_ptr(torch, stream))
    _raise_for(rc, "lbkd_build_rr_host", n, k)


def host_join(*, device: int = 0, stream=None, sync: bool = True) -> None:
    """Wait for every pipelined host build (lbkd_host_join); raises the
    reference's ValueError if any of their inputs was non-finite."""
    torch = _torch()
    lib = _native.load()
    with torch.cuda.device(device):
        rc = lib.lbkd_host_join(_native.context(device), _stream_ptr(torch, stream), 1 if sync else 0)
    _raise_for(rc, "lbkd_host_join", 0, 0)


def _raise_for(rc: int, where: str, n: int, k: int, widest: bool = False) -> None:
    if rc == _native.LBKD_OK:
        return
    if rc == _native.LBKD_ENONFINITE:
        raise ValueError("coordinates must be finite (no NaN or infinity)")
    if rc == _native.LBKD_ECAPACITY:
        if widest:
            raise ValueError(f"{n} points with {k} dimensions exceed the 32-bit tag capacity")
        raise ValueError(f"{n} points exceed the 32-bit tag capacity ({MAX_POINTS})")
    raise _native.NativeError(rc, where)


def last_launch_count(device: int = 0) -> int:
    lib = _native.load()
    return int(lib.lbkd_last_launch_count(_native.context(device)))


def _record_trace(recorder, pts, out, perm, trace, n, k, tags_of_node=None):
    """Rebuild the reference's per-phase (tags, coords) arrays (builder.py:
    219-235) from the device trace: after sort l the array is the finalized
    nodes 0..F(l)-1 in node order followed by W_l, the traced order."""
    L = treemath.num_levels(n)
    pack = tags_of_node if tags_of_node is not None else (lambda nodes: nodes.astype(np.uint32))
    tags0 = pack(np.zeros(n, dtype=np.int64))
    recorder.tags_allocated(np.zeros(n, dtype=np.uint32))
    recorder.phase("init", -1, tags0, pts.astype(np.float64))
    for l in range(L - 1):
        top = (1 << l) - 1
        rows = np.concatenate([perm[:top].astype(np.int64), trace[l, : n - top].astype(np.int64)])
        sizes = treemath.segment_sizes(n, l)
        seg_nodes = np.repeat(np.arange(top, top + len(sizes), dtype=np.int64), sizes)
        tags = np.concatenate([np.arange(top, dtype=np.int64), seg_nodes])
        recorder.phase("sort", l, pack(tags), pts[rows].astype(np.float64))
        # update pass l (kernels_numpy.py:41-48)
        upd = tags.copy()
        start = top
        for j, sz in enumerate(sizes):
            s = top + j
            piv_off = treemath.pivot_pos(s, n) - treemath.segment_begin(s, n)
            seg = np.arange(sz)
            upd[start:start + sz] = np.where(seg < piv_off, 2 * s + 1, np.where(seg > piv_off, 2 * s + 2, s))
            start += sz
        recorder.phase("update", l, pack(upd), pts[rows].astype(np.float64))
    recorder.phase("sort", L - 1, pack(np.arange(n, dtype=np.int64)), out.astype(np.float64))


def build_round_robin(points, k: int | None = None, payload=None, *, skip_prefix: bool = False,
                      recorder: BuildRecorder | None = None) -> KdTree:
    """Drop-in for lbkd.build_round_robin (builder.py:200-236).

    ``skip_prefix`` is accepted for signature compatibility; the result is
    identical either way (the GPU path never re-sorts finalized nodes).
    """
    coords, payload = ingest(points, k, payload)
    n = coords.shape[0]
    kd = coords.shape[1] if coords.ndim == 2 else 1
    if n == 0:
        if recorder is not None:
            recorder.tags_allocated(np.zeros(0, dtype=np.uint32))
        return KdTree(coords.astype(np.float64), payload)
    torch = _torch()
    capture = recorder is not None and recorder.capture
    dev = torch.cuda.current_device()
    d_pts = torch.from_numpy(coords).to(device=f"cuda:{dev}")
    trace = None
    if capture:
        cap = int(_native.load().lbkd_single_cta_capacity(kd, 0))
        if n > cap:
            raise ValueError(f"BuildRecorder(capture=True) is supported for n <= {cap}")
        L = treemath.num_levels(n)
        trace = torch.zeros(max(L, 1) * n, dtype=torch.int32, device=d_pts.device)
    out, perm = build_round_robin_cuda(d_pts, trace=trace)
    out_h = out.cpu().numpy()
    perm_h = perm.cpu().numpy().view(np.uint32).astype(np.int64)
    if recorder is not None:
        if capture:
            tr = trace.cpu().numpy().view(np.uint32).reshape(-1, n)
            _record_trace(recorder, coords, out_h, perm_h, tr, n, kd)
        else:
            L = treemath.num_levels(n)
            recorder.tags_allocated(np.zeros(n, dtype=np.uint32))
            recorder.sort_phases += L
            recorder.update_phases += L - 1
    return KdTree(out_h.astype(np.float64), payload[perm_h])
