"""CPU-only checks of the C-ABI library and host logic (no compute calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2211_00120_b200 import _native, build_native, treemath
from paper_2211_00120_b200.builder import ingest
from paper_2211_00120_b200.widest import dim_bits_for, pack_tag, unpack_tag, widest_dim, world_bounds
from oracle import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "lbkd_b200.h")).read()
    return sorted(set(re.findall(r"\b(lbkd_[a-z_0-9]+)\s*\(", text)))


def test_library_builds_and_exports_every_header_symbol():
    path = build_native.build()
    lib = ctypes.CDLL(path)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTED)


def test_host_helpers_in_library():
    lib = _native.load()
    for n in (1, 2, 3, 10, 1000, 10**8, 2**31 - 1):
        assert lib.lbkd_num_levels(n) == treemath.num_levels(n)
    assert lib.lbkd_strerror(2).decode().startswith("coordinates must be finite")
    # the chosen geometry keeps a tile inside at most two segments
    for n in (10, 8191, 8192, 10**6, 10**8, 10**9):
        for k in (1, 2, 3, 4, 5, 8, 16):
            for w in (False, True):
                b, lam0 = _native.plan_info(n, k, w)
                L = n.bit_length()
                assert lam0 == max(0, L - b)
                if lam0 > 0:
                    min_seg = (1 << (L - (lam0 - 1) - 1)) - 1
                    assert (1 << (b - 1)) <= min_seg
                assert (1 << (L - lam0)) - 1 <= (1 << b) - 1  # subtree fits a CTA


def test_treemath_mirror_matches_oracle_restatement():
    for n in range(1, 600):
        for s in range(n):
            assert treemath.subtree_size(s, n) == oracle.subtree_size(s, n)
            assert treemath.segment_begin(s, n) == oracle.segment_begin(s, n)


def test_treemath_hand_values():
    # reference tests/test_treemath.py hand tables (n = 10 walkthrough tree)
    assert [treemath.subtree_size(s, 10) for s in range(10)] == [10, 6, 3, 3, 2, 1, 1, 1, 1, 1]
    assert treemath.pivot_pos(0, 10) == 6
    assert treemath.segment_begin(2, 10) == 7
    assert treemath.segment_sizes(10, 1) == [6, 3]


def test_ingest_contract():
    with pytest.raises(ValueError):
        ingest(np.array([[1.0], [np.nan]]))
    with pytest.raises(ValueError):
        ingest(np.array([[1.0], [np.inf]]))
    with pytest.raises(ValueError):
        ingest(np.zeros((3, 2, 2)))
    with pytest.raises(ValueError):
        ingest(np.zeros((4, 3)), 2)
    with pytest.raises(ValueError):
        ingest(np.zeros((4, 0)))
    with pytest.raises(ValueError):
        ingest(np.zeros((4, 1)), 1, payload=np.arange(3))
    with pytest.raises(ValueError):
        ingest(np.broadcast_to(np.zeros((1, 1)), (2**31, 1)))
    # float64 input is accepted like the reference's: float32-exact values take
    # the float32 device path, anything else the float64 one
    c, _ = ingest(np.array([[0.1]], dtype=np.float64))
    assert c.dtype == np.float64 and c[0, 0] == 0.1
    c, _ = ingest(np.array([[1e300], [-0.0]]))
    assert c.dtype == np.float64
    c, _ = ingest(np.array([[0.5, -0.0], [3.0, 1e-3]]).astype(np.float32).astype(np.float64))
    assert c.dtype == np.float32 and np.signbit(c[0, 1])
    c, p = ingest([5.0, 1.0, 9.0])
    assert c.dtype == np.float32 and c.shape == (3, 1) and p.tolist() == [0, 1, 2]


def test_widest_host_helpers():
    assert [dim_bits_for(k) for k in (1, 2, 3, 4, 5)] == [0, 1, 2, 2, 3]
    for bits in (0, 1, 2, 3):
        for node in (0, 5, 1000):
            for dim in range(max(1 << bits, 1)):
                assert unpack_tag(pack_tag(node, dim, bits), bits) == (node, dim)
    box = world_bounds(np.array([[0.0, 5.0], [4.0, 5.0], [2.0, 11.0]]))
    assert widest_dim(box) == 1
    assert widest_dim(world_bounds(np.array([[0.0, 0.0], [3.0, 3.0]]))) == 0


def test_flip_key_restatement_orders_like_numpy():
    # the device key: order-flipped float32 bits with -0.0 canonicalised
    vals = np.array([-np.inf, -3.5, -1e-30, -0.0, 0.0, 1e-38, 2.0, np.inf], dtype=np.float32)
    u = vals.view(np.uint32).copy()
    u[u == 0x80000000] = 0
    key = np.where(u >> 31, ~u, u | 0x80000000).astype(np.uint32)
    assert np.all(np.diff(key.astype(np.int64)) >= 0)
    assert key[3] == key[4]


def test_entry_points_fail_loudly_without_cuda():
    """No CPU fallback: every build entry point raises when no CUDA device is
    present (here), before any work -- including the pipelined host-buffer
    variants."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    import paper_2211_00120_b200 as kd
    from paper_2211_00120_b200.builder import build_round_robin_host

    pts = np.random.default_rng(0).random((100, 3), dtype=np.float32)
    t = torch.from_numpy(pts)
    out = torch.empty_like(t)
    perm = torch.empty(100, dtype=torch.int32)
    dims = torch.empty(100, dtype=torch.uint8)
    calls = [
        lambda: kd.build_round_robin(pts),
        lambda: kd.build_widest(pts),
        lambda: build_round_robin_host(t, out, perm),
        lambda: kd.build_widest_host(t, out, perm, dims),
    ]
    for call in calls:
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            call()
