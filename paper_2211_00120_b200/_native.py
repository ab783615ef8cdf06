"""ctypes binding of the in-tree C-ABI library (include/lbkd_b200.h).

There is exactly one backend: the sm_100a CUDA library.  If it is missing or
no CUDA device is present the build entry points raise -- there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "liblbkd_b200.so")

LBKD_OK = 0
LBKD_EINVAL_SHAPE = 1
LBKD_ENONFINITE = 2
LBKD_ECAPACITY = 3
LBKD_ECUDA = 4
LBKD_ENOPEER = 5
LBKD_ENOMEM = 6
LBKD_EUNSUPPORTED = 7

EXPORTED = (
    "lbkd_create", "lbkd_destroy", "lbkd_set_check",
    "lbkd_build_rr", "lbkd_build_widest",
    "lbkd_build_rr_trace", "lbkd_build_widest_trace",
    "lbkd_build_rr_f64", "lbkd_build_widest_f64", "lbkd_build_rr_f64_trace", "lbkd_build_widest_f64_trace",
    "lbkd_update_tags_rr", "lbkd_update_tags_widest",
    "lbkd_num_levels", "lbkd_single_cta_capacity", "lbkd_plan_info",
    "lbkd_last_launch_count", "lbkd_strerror", "lbkd_last_cuda_error",
    "lbkd_set_profile", "lbkd_profile_read",
    "lbkd_build_rr_top", "lbkd_build_rr_sub", "lbkd_build_rr_split",
    "lbkd_profile_kernel", "lbkd_set_algorithm", "lbkd_get_algorithm", "lbkd_set_level_pairs",
    "lbkd_build_rr_host", "lbkd_build_widest_host", "lbkd_host_join",
    "lbkd_set_subtree_kernel",
    "lbkd_knn", "lbkd_radius_count", "lbkd_radius_scratch_len", "lbkd_radius_fill",
    "lbkd_check_valid", "lbkd_subtree_boxes",
    "lbkd_knn_f64", "lbkd_radius_count_f64", "lbkd_radius_fill_f64", "lbkd_check_valid_f64",
    "lbkd_subtree_boxes_f64",
)

# kernel classes of lbkd_profile_kernel
PROFILE_CLASSES = ("init", "hist", "pick", "filter", "select", "partition", "subtree", "sort_pass", "other")
ALGORITHMS = ("select", "sort")

_lib = None
_lock = threading.Lock()
_ctxs: dict = {}


class NativeError(RuntimeError):
    def __init__(self, code: int, where: str):
        lib = load()
        msg = lib.lbkd_strerror(code).decode()
        if code == LBKD_ECUDA:
            msg += ": " + lib.lbkd_last_cuda_error().decode()
        super().__init__(f"{where}: {msg} (code {code})")
        self.code = code


def load():
    """Load the library (building it first if this checkout has none)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            from . import build_native
            build_native.build()
        lib = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.lbkd_create.argtypes = [ctypes.POINTER(vp), i32]
        lib.lbkd_create.restype = i32
        lib.lbkd_destroy.argtypes = [vp]
        lib.lbkd_destroy.restype = None
        lib.lbkd_set_check.argtypes = [vp, i32]
        lib.lbkd_set_check.restype = None
        lib.lbkd_build_rr.argtypes = [vp, vp, vp, i64, i32, vp, vp]
        lib.lbkd_build_rr.restype = i32
        lib.lbkd_build_widest.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp]
        lib.lbkd_build_widest.restype = i32
        lib.lbkd_build_rr_trace.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp]
        lib.lbkd_build_rr_trace.restype = i32
        lib.lbkd_build_widest_trace.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp, vp]
        lib.lbkd_build_widest_trace.restype = i32
        lib.lbkd_build_rr_f64.argtypes = [vp, vp, vp, i64, i32, vp, vp]
        lib.lbkd_build_rr_f64.restype = i32
        lib.lbkd_build_widest_f64.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp]
        lib.lbkd_build_widest_f64.restype = i32
        lib.lbkd_build_rr_f64_trace.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp]
        lib.lbkd_build_rr_f64_trace.restype = i32
        lib.lbkd_build_widest_f64_trace.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp, vp]
        lib.lbkd_build_widest_f64_trace.restype = i32
        lib.lbkd_build_rr_top.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp, i64, vp]
        lib.lbkd_build_rr_top.restype = i32
        lib.lbkd_build_rr_sub.argtypes = [vp, vp, i64, i64, i32, i32, i64, vp, vp, vp]
        lib.lbkd_build_rr_sub.restype = i32
        lib.lbkd_build_rr_split.argtypes = [vp, vp, vp, i64, i64, i32, i32, i64, vp, vp, vp, vp]
        lib.lbkd_build_rr_split.restype = i32
        lib.lbkd_update_tags_rr.argtypes = [vp, i64, i32, i32, vp]
        lib.lbkd_update_tags_rr.restype = i32
        lib.lbkd_update_tags_widest.argtypes = [vp, vp, i32, vp, vp, vp, i64, i32, i32, i32, vp]
        lib.lbkd_update_tags_widest.restype = i32
        lib.lbkd_num_levels.argtypes = [i64]
        lib.lbkd_num_levels.restype = i32
        lib.lbkd_single_cta_capacity.argtypes = [i32, i32]
        lib.lbkd_single_cta_capacity.restype = i64
        lib.lbkd_plan_info.argtypes = [i64, i32, i32, ctypes.POINTER(i32), ctypes.POINTER(i32)]
        lib.lbkd_plan_info.restype = i32
        lib.lbkd_last_launch_count.argtypes = [vp]
        lib.lbkd_last_launch_count.restype = i64
        lib.lbkd_set_profile.argtypes = [vp, i32]
        lib.lbkd_set_profile.restype = None
        dp = ctypes.POINTER(ctypes.c_double)
        lib.lbkd_profile_read.argtypes = [vp, ctypes.POINTER(i32), dp, dp]
        lib.lbkd_profile_read.restype = i32
        lib.lbkd_profile_kernel.argtypes = [vp, i32, ctypes.POINTER(i32), dp, dp]
        lib.lbkd_profile_kernel.restype = i32
        lib.lbkd_set_algorithm.argtypes = [vp, i32]
        lib.lbkd_set_algorithm.restype = i32
        lib.lbkd_get_algorithm.argtypes = [vp]
        lib.lbkd_get_algorithm.restype = i32
        lib.lbkd_set_level_pairs.argtypes = [vp, i32]
        lib.lbkd_set_level_pairs.restype = i32
        lib.lbkd_build_rr_host.argtypes = [vp, vp, vp, i64, i32, vp, vp]
        lib.lbkd_build_rr_host.restype = i32
        lib.lbkd_build_widest_host.argtypes = [vp, vp, vp, i64, i32, vp, vp, vp]
        lib.lbkd_build_widest_host.restype = i32
        lib.lbkd_host_join.argtypes = [vp, vp, i32]
        lib.lbkd_host_join.restype = i32
        lib.lbkd_set_subtree_kernel.argtypes = [vp, i32]
        lib.lbkd_set_subtree_kernel.restype = i32
        f64 = ctypes.c_double
        lib.lbkd_knn.argtypes = [vp, i64, i32, vp, vp, i64, i32, vp, vp, vp]
        lib.lbkd_knn.restype = i32
        lib.lbkd_radius_count.argtypes = [vp, i64, i32, vp, vp, i64, f64, vp, vp, vp, vp]
        lib.lbkd_radius_count.restype = i32
        lib.lbkd_radius_scratch_len.argtypes = [i64]
        lib.lbkd_radius_scratch_len.restype = i64
        lib.lbkd_radius_fill.argtypes = [vp, i64, i32, vp, vp, i64, f64, vp, vp, vp]
        lib.lbkd_radius_fill.restype = i32
        lib.lbkd_check_valid.argtypes = [vp, i64, i32, vp, vp, vp, vp]
        lib.lbkd_check_valid.restype = i32
        lib.lbkd_subtree_boxes.argtypes = [vp, i64, i32, vp, vp, vp, vp]
        lib.lbkd_subtree_boxes.restype = i32
        for suffix in ("", "_f64"):
            getattr(lib, "lbkd_knn" + suffix).argtypes = [vp, i64, i32, vp, vp, i64, i32, vp, vp, vp]
            getattr(lib, "lbkd_knn" + suffix).restype = i32
            getattr(lib, "lbkd_radius_count" + suffix).argtypes = [vp, i64, i32, vp, vp, i64, f64, vp, vp, vp, vp]
            getattr(lib, "lbkd_radius_count" + suffix).restype = i32
            getattr(lib, "lbkd_radius_fill" + suffix).argtypes = [vp, i64, i32, vp, vp, i64, f64, vp, vp, vp]
            getattr(lib, "lbkd_radius_fill" + suffix).restype = i32
            getattr(lib, "lbkd_check_valid" + suffix).argtypes = [vp, i64, i32, vp, vp, vp, vp]
            getattr(lib, "lbkd_check_valid" + suffix).restype = i32
            getattr(lib, "lbkd_subtree_boxes" + suffix).argtypes = [vp, i64, i32, vp, vp, vp, vp]
            getattr(lib, "lbkd_subtree_boxes" + suffix).restype = i32
        lib.lbkd_strerror.argtypes = [i32]
        lib.lbkd_strerror.restype = ctypes.c_char_p
        lib.lbkd_last_cuda_error.argtypes = []
        lib.lbkd_last_cuda_error.restype = ctypes.c_char_p
        _lib = lib
        return lib


def context(device: int):
    """One lbkd_ctx per (thread, device); contexts own the scratch buffers."""
    key = (threading.get_ident(), int(device))
    ctx = _ctxs.get(key)
    if ctx is None:
        lib = load()
        p = ctypes.c_void_p()
        rc = lib.lbkd_create(ctypes.byref(p), int(device))
        if rc != LBKD_OK:
            raise NativeError(rc, "lbkd_create")
        ctx = p
        _ctxs[key] = ctx
    return ctx


def check(rc: int, where: str) -> None:
    if rc != LBKD_OK:
        raise NativeError(rc, where)


def profile_read(device: int = 0):
    """(digit-pass launches, their device ms, their algorithmic bytes) of the
    last build on this thread's context for `device` (lbkd_set_profile on)."""
    lib = load()
    n = ctypes.c_int()
    ms = ctypes.c_double()
    by = ctypes.c_double()
    check(lib.lbkd_profile_read(context(device), ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by)), "lbkd_profile_read")
    return n.value, ms.value, by.value


def profile_kernels(device: int = 0) -> dict:
    """{class: (launches, device ms, algorithmic bytes)} of the last profiled
    build on this thread's context for `device`."""
    lib = load()
    out = {}
    for i, name in enumerate(PROFILE_CLASSES):
        n = ctypes.c_int()
        ms = ctypes.c_double()
        by = ctypes.c_double()
        check(lib.lbkd_profile_kernel(context(device), i, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(by)),
              "lbkd_profile_kernel")
        if n.value:
            out[name] = (n.value, ms.value, by.value)
    return out


def set_algorithm(algo: str, device: int = 0) -> None:
    """Global-level algorithm of this thread's context: "select" (pivot
    selection + stable partition, default) or "sort" (per-level radix sort)."""
    check(load().lbkd_set_algorithm(context(device), ALGORITHMS.index(algo)), "lbkd_set_algorithm")


def set_level_pairs(on: bool, device: int = 0) -> None:
    """Round robin: two global levels per partition pass (default) or one."""
    check(load().lbkd_set_level_pairs(context(device), 1 if on else 0), "lbkd_set_level_pairs")


def set_subtree_kernel(which: str, device: int = 0) -> None:
    """In-CTA phase of this thread's context: "default", "lists" or "selection"."""
    code = {"default": -1, "lists": 0, "selection": 1}[which]
    check(load().lbkd_set_subtree_kernel(context(device), code), "lbkd_set_subtree_kernel")


def get_algorithm(device: int = 0) -> str:
    return ALGORITHMS[load().lbkd_get_algorithm(context(device))]


def set_profile(on: bool, device: int = 0) -> None:
    load().lbkd_set_profile(context(device), 1 if on else 0)


def plan_info(n: int, k: int, widest: bool):
    lib = load()
    b = ctypes.c_int()
    lam0 = ctypes.c_int()
    check(lib.lbkd_plan_info(int(n), int(k), int(widest), ctypes.byref(b), ctypes.byref(lam0)), "lbkd_plan_info")
    return b.value, lam0.value
