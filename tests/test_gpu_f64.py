"""float64 input -- the reference's own dtype (ingest promotes everything to
float64, /root/reference/pkg/src/lbkd/builder.py:131-133).

The drop-in sends float64 input that is not float32-representable through
lbkd_build_*_f64 (csrc/rank64.cu: per-dimension dense ranks coded as
float32, the float32 build, float64 rows gathered by the permutation; widest
widths from a table of the original values).  Pinned against the reference's
own outputs (tests/golden/hashes_f64.json, tests/golden/make_golden_f64.py)
and, at larger sizes, against the recursive oracle's float64 instantiation.
"""

import ctypes
import hashlib

import numpy as np
import pytest

from oracle import oracle
from tests.golden_util import f64_cases, gen_f64

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import _native, queries, verify  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("case", f64_cases(), ids=lambda c: f"{c['mode']}-{c['kind']}-{c['n']}-k{c['k']}")
def test_reference_hashes_float64(case):
    pts = gen_f64(case["kind"], case["n"], case["k"], case["seed"])
    assert sha(pts) == case["input_sha256"]
    if case["mode"] == "rr":
        tree = kd.build_round_robin(pts)
        assert tree.split_dims is None
    else:
        tree = kd.build_widest(pts)
        assert sha(tree.split_dims.astype(np.uint8)) == case["split_dims_sha256"]
    assert tree.coords.dtype == np.float64 and tree.payload.dtype == np.int64
    assert tree.payload[:32].tolist() == case["perm_head"]
    assert sha(tree.payload.astype(np.uint32)) == case["perm_sha256"]
    assert sha(tree.coords) == case["coords_sha256"]


@pytest.mark.parametrize("kind", ["uniform64", "clustered64", "ties64", "near64", "range64", "signed_zero64"])
def test_device_float64_against_oracle(kind):
    n, k = 3_000_017, 3
    pts = gen_f64(kind, n, k, seed=42)
    d = torch.from_numpy(pts).cuda()
    out, perm = kd.build_round_robin_cuda(d)
    assert out.dtype == torch.float64
    want = oracle.rec_build(pts)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), want)
    assert np.array_equal(out.cpu().numpy().view(np.uint64), pts[want.astype(np.int64)].view(np.uint64))
    out, perm, dims = kd.build_widest_cuda(d)
    wp, wd = oracle.rec_build(pts, widest=True)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), wp)
    assert np.array_equal(dims.cpu().numpy(), wd)


def test_float64_reference_bench_config():
    """The reference's own bench input (cli.py:176-177: default_rng(0).random
    ((10M, 4)), float64) at the size of BASELINE config 3."""
    pts = np.random.default_rng(0).random((10_000_000, 4))
    _, perm = kd.build_round_robin_cuda(torch.from_numpy(pts).cuda())
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(pts))


def test_float64_in_place_and_small_sizes():
    for n in (1, 2, 3, 31, 1000, 4095, 4096, 70_001):
        pts = gen_f64("uniform64", n, 3, seed=n)
        d = torch.from_numpy(pts).cuda()
        want = oracle.rec_build(pts)
        _, perm = kd.build_round_robin_cuda(d, out=d)  # in place
        assert np.array_equal(perm.cpu().numpy().view(np.uint32), want), n
        assert np.array_equal(d.cpu().numpy(), pts[want.astype(np.int64)]), n


def test_float64_nonfinite_and_recorder():
    lib = _native.load()
    ctx = _native.context(0)
    for n in (5, 100_000):
        p = gen_f64("uniform64", n, 2, seed=1)
        p[n // 3, 1] = np.inf
        d = torch.from_numpy(p).cuda()
        out = torch.empty_like(d)
        perm = torch.empty(n, dtype=torch.int32, device="cuda")
        lib.lbkd_set_check(ctx, 1)
        rc = lib.lbkd_build_rr_f64(ctx, d.data_ptr(), out.data_ptr(), n, 2, perm.data_ptr(),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == _native.LBKD_ENONFINITE
    with pytest.raises(ValueError, match="finite"):
        kd.build_round_robin(np.array([[0.1], [np.nan]]))
    # BuildRecorder(capture=True) on float64 input: every snapshot holds the
    # float64 rows of the traced order; the final one is the tree
    pts = gen_f64("ties64", 3000, 3, seed=5)
    rec = kd.BuildRecorder(capture=True)
    tree = kd.build_round_robin(pts, recorder=rec)
    assert rec.sort_phases == 12 and rec.update_phases == 11
    assert np.array_equal(rec.snapshots[-1].coords, tree.coords)
    assert np.array_equal(tree.payload, oracle.rec_build(pts).astype(np.int64))


def test_queries_and_validation_on_float64_trees():
    pts = gen_f64("clustered64", 20_000, 3, seed=3)
    for build in (kd.build_round_robin, kd.build_widest):
        tree = build(pts)
        assert verify.check_valid(tree).valid
        q = gen_f64("clustered64", 64, 3, seed=4)
        for i in range(0, 64, 7):
            got = queries.knn(tree, q[i], 5)
            want = oracle.brute_knn(tree.coords, q[i], 5)
            assert [(g.index, g.dist2) for g in got] == [(int(a), float(b)) for a, b in want]
            r = queries.radius_query(tree, q[i], 0.02)
            assert r.tolist() == sorted(oracle.brute_radius(tree.coords, q[i], 0.02).tolist())
        lo, hi = verify.brute_subtree_boxes(tree)
        wlo, whi = oracle.brute_subtree_boxes(tree.coords, tree.split_dims)
        assert np.array_equal(lo, wlo) and np.array_equal(hi, whi)
    tree.coords[3, 0] = 1e9  # an in-place edit breaks the ordering
    assert not verify.check_valid(tree).valid
