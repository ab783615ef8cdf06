"""GPU robustness: adversarial inputs against the oracle, and the contracts
of the C ABI that the round-1 review found broken (host-pipeline regrowth,
builds sharing one context's scratch across streams, the non-finite flag of
single-CTA builds, stale query caches, caller-buffer validation).

Oracle: oracle.rec_build (oracle/lbkd_recursive.cpp, the threaded
restatement of verify.reference_build, pinned to the reference's own hashes
in tests/test_oracle.py)."""

import ctypes

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import _native, datagen  # noqa: E402


def _adversarial(name, n, k, seed):
    rng = np.random.default_rng(seed)
    if name == "identical":
        return np.full((n, k), 0.25, np.float32)
    if name == "identical_zero_signs":  # -0.0 and +0.0 only: all ties
        return np.where(rng.random((n, k)) < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32)
    if name == "huge_range":
        return (10.0 ** rng.uniform(-30, 30, (n, k)) * np.where(rng.random((n, k)) < 0.5, -1, 1)).astype(np.float32)
    if name == "constant_axis":
        p = datagen.uniform(n, k, seed)
        p[:, k // 2] = 7.0
        return p
    if name == "sorted":
        return np.sort(datagen.uniform(n, k, seed), axis=0)
    if name == "reverse_sorted":
        return np.sort(datagen.uniform(n, k, seed), axis=0)[::-1].copy()
    if name == "two_values":
        return rng.integers(0, 2, size=(n, k)).astype(np.float32)
    if name == "denormals":
        return (rng.integers(-1000, 1000, size=(n, k)).astype(np.float32) * np.float32(1e-42)).astype(np.float32)
    if name == "one_hot_line":  # all points on a line: ties in every other dim
        t = rng.random(n, dtype=np.float32)
        p = np.zeros((n, k), np.float32)
        p[:, 0] = t
        return p
    raise ValueError(name)


ADVERSARIAL = ["identical", "identical_zero_signs", "huge_range", "constant_axis", "sorted", "reverse_sorted",
               "two_values", "denormals", "one_hot_line"]


def _dev(p):
    return torch.from_numpy(np.ascontiguousarray(p)).cuda()


@pytest.mark.parametrize("name", ADVERSARIAL)
@pytest.mark.parametrize("n,k", [(2_000_003, 3), (700_001, 2)])
def test_adversarial_rr(name, n, k):
    pts = _adversarial(name, n, k, seed=n % 97)
    out, perm = kd.build_round_robin_cuda(_dev(pts))
    want = oracle.rec_build(pts)
    got = perm.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want), name
    assert np.array_equal(out.cpu().numpy().view(np.uint32), pts[want.astype(np.int64)].view(np.uint32))


@pytest.mark.parametrize("name", ADVERSARIAL)
@pytest.mark.parametrize("n,k", [(2_000_003, 3), (300_001, 4)])
def test_adversarial_widest(name, n, k):
    pts = _adversarial(name, n, k, seed=n % 89)
    out, perm, dims = kd.build_widest_cuda(_dev(pts))
    wp, wd = oracle.rec_build(pts, widest=True)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), wp), name
    assert np.array_equal(dims.cpu().numpy(), wd), name


@pytest.mark.parametrize("name", ["identical", "huge_range", "constant_axis", "sorted"])
def test_adversarial_10m(name):
    pts = _adversarial(name, 10_000_000, 3, seed=3)
    _, perm = kd.build_round_robin_cuda(_dev(pts))
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(pts)), name
    _, perm, dims = kd.build_widest_cuda(_dev(pts))
    wp, wd = oracle.rec_build(pts, widest=True)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), wp), name
    assert np.array_equal(dims.cpu().numpy(), wd), name


@pytest.mark.parametrize("pairs", [True, False])
@pytest.mark.parametrize("name", ["identical", "huge_range", "constant_axis", "two_values", "one_hot_line", "sorted"])
def test_level_pairs_both_schedules(name, pairs):
    """Round robin with the global levels two per partition pass (default:
    the second level selected in the first's layout -- identical children
    keyed by their index column) and one per pass: both exact, for odd and
    even numbers of global levels and k = 2, 3, 4."""
    _native.set_level_pairs(pairs)
    try:
        for n, k in ((1_500_001, 3), (2_500_001, 2), (600_001, 4)):
            pts = _adversarial(name, n, k, seed=n % 91)
            _, perm = kd.build_round_robin_cuda(_dev(pts))
            assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(pts)), (name, n, k)
    finally:
        _native.set_level_pairs(True)


@pytest.mark.parametrize("dim", [0, 1, 2])
def test_nonfinite_input_is_reported_not_crashing(dim):
    """NaN / inf rows in a multi-level build (the level-pair kernels, the
    partitions, the in-CTA kernels) end in the ValueError of
    builder.py:134-135 -- never a device fault -- and the context keeps
    working."""
    pts = datagen.uniform(700_001, 3, seed=dim)
    bad = pts.copy()
    bad[::9973, dim] = np.nan
    bad[5, (dim + 1) % 3] = np.inf
    for fn in (kd.build_round_robin_cuda, kd.build_widest_cuda):
        with pytest.raises(ValueError, match="finite"):
            fn(_dev(bad))
    _, perm = kd.build_round_robin_cuda(_dev(pts))
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(pts))


_WIDEST_PAIRS = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2211_00120_b200 as kd
from oracle import oracle
from tests.test_gpu_robust import _adversarial
from paper_2211_00120_b200 import datagen
cases = [("uniform", datagen.uniform(1_500_001, 3, 1)), ("clustered", datagen.make("clustered", 600_001, 2, 2)),
         ("ties", datagen.ties(1_000_003, 4, 3))]
cases += [(nm, _adversarial(nm, 700_001, 3, 5)) for nm in ("identical", "huge_range", "constant_axis", "sorted")]
for name, p in cases:
    _, perm, dims = kd.build_widest_cuda(torch.from_numpy(np.ascontiguousarray(p)).cuda())
    wp, wd = oracle.rec_build(p, widest=True)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), wp), name
    assert np.array_equal(dims.cpu().numpy(), wd), name
print("WIDEST_PAIRS_OK")
'''


def test_widest_level_pairs_opt_in():
    """Widest with its global levels two per partition pass (off by default:
    measured slower on config 5; LBKD_PAIR_WIDEST=1): exact on normal and
    adversarial inputs, odd and even level counts, k = 2, 3, 4."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LBKD_PAIR_WIDEST="1")
    r = subprocess.run([sys.executable, "-c", _WIDEST_PAIRS, root], env=env, cwd=root, capture_output=True,
                       text=True, timeout=900)
    assert "WIDEST_PAIRS_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_ties_100m_rr():
    """64 values per axis at the headline size (ties at every level)."""
    pts = datagen.ties(100_000_000, 3, seed=1)
    _, perm = kd.build_round_robin_cuda(_dev(pts))
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(pts))


# --- C-ABI contracts ---------------------------------------------------------

def test_host_pipeline_regrows_on_n_not_only_n_times_k():
    """a later host build with more points and fewer
    dimensions (n*k within capacity, n beyond it) must not overrun the
    perm / split-dim buffers."""
    from paper_2211_00120_b200.builder import build_round_robin_host, host_join
    from paper_2211_00120_b200.widest import build_widest_host

    shapes = [(1000, 4), (3001, 1), (50_000, 8), (390_000, 1), (100_003, 3)]
    res = []
    for i, (n, k) in enumerate(shapes):
        p = datagen.uniform(n, k, seed=i)
        hin = torch.from_numpy(p).pin_memory()
        hout = torch.empty((n, k), dtype=torch.float32).pin_memory()
        hperm = torch.empty(n, dtype=torch.int32).pin_memory()
        hdims = torch.empty(n, dtype=torch.uint8).pin_memory()
        if i % 2:
            build_widest_host(hin, hout, hperm, hdims)
        else:
            build_round_robin_host(hin, hout, hperm)
        res.append((p, hout, hperm, hdims, i % 2))
    host_join()
    for p, hout, hperm, hdims, widest in res:
        if widest:
            wp, wd = oracle.rec_build(p, widest=True)
            assert np.array_equal(hperm.numpy().view(np.uint32), wp)
            assert np.array_equal(hdims.numpy(), wd)
        else:
            wp = oracle.rec_build(p)
            assert np.array_equal(hperm.numpy().view(np.uint32), wp)
        assert np.array_equal(hout.numpy(), p[wp.astype(np.int64)])


def test_device_build_after_host_builds_on_other_stream():
    """host-pipeline builds and device builds share the
    context's scratch; a device build enqueued on another stream right after
    pipelined host builds (no join in between) must wait for them."""
    from paper_2211_00120_b200.builder import build_round_robin_host, host_join

    n, k = 3_000_001, 3
    inputs = [datagen.make(kind, n, k, seed=s) for s, kind in enumerate(("uniform", "clustered", "ties"))]
    hin = [torch.from_numpy(p).pin_memory() for p in inputs]
    hout = [torch.empty((n, k), dtype=torch.float32).pin_memory() for _ in inputs]
    hperm = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in inputs]
    dev_pts = _dev(datagen.clustered(n, k, seed=9))
    side = torch.cuda.Stream()
    for rep in range(2):
        for i in range(len(inputs)):
            build_round_robin_host(hin[i], hout[i], hperm[i])
        with torch.cuda.stream(side):
            out, perm = kd.build_round_robin_cuda(dev_pts, stream=side, check_finite=False)
        side.synchronize()
        host_join()
        assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(dev_pts.cpu().numpy())), rep
        for i, p in enumerate(inputs):
            assert np.array_equal(hperm[i].numpy().view(np.uint32), oracle.rec_build(p)), (rep, i)


def test_host_nonfinite_flag_does_not_blame_device_builds():
    """A NaN in a pipelined host build is reported by host_join only; a
    device build in between (check on) still succeeds."""
    from paper_2211_00120_b200.builder import build_round_robin_host, host_join

    n, k = 200_003, 3
    bad = datagen.uniform(n, k, seed=2)
    bad[11, 2] = np.nan
    hb = torch.from_numpy(bad).pin_memory()
    hout = torch.empty((n, k), dtype=torch.float32).pin_memory()
    hperm = torch.empty(n, dtype=torch.int32).pin_memory()
    build_round_robin_host(hb, hout, hperm)
    good = datagen.uniform(n, k, seed=3)
    _, perm = kd.build_round_robin_cuda(_dev(good))  # check_finite=True
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(good))
    with pytest.raises(ValueError, match="finite"):
        host_join()


@pytest.mark.parametrize("n", [1, 2, 7, 100, 4000])
def test_single_cta_builds_report_nonfinite(n):
    """Builds without global levels read the caller's array directly; the C
    ABI must still report non-finite input (builder.py:134-135)."""
    lib = _native.load()
    ctx = _native.context(0)
    for mode in ("rr", "widest"):
        for val in (np.nan, np.inf, -np.inf):
            p = datagen.uniform(n, 3, seed=n)
            p[n // 2, 1] = val
            d = _dev(p)
            out = torch.empty_like(d)
            perm = torch.empty(n, dtype=torch.int32, device="cuda")
            dims = torch.empty(n, dtype=torch.uint8, device="cuda")
            lib.lbkd_set_check(ctx, 1)
            s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            if mode == "rr":
                rc = lib.lbkd_build_rr(ctx, d.data_ptr(), out.data_ptr(), n, 3, perm.data_ptr(), s)
            else:
                rc = lib.lbkd_build_widest(ctx, d.data_ptr(), out.data_ptr(), n, 3, perm.data_ptr(),
                                           dims.data_ptr(), s)
            assert rc == _native.LBKD_ENONFINITE, (mode, val, rc)
            with pytest.raises(ValueError, match="finite"):
                (kd.build_round_robin_cuda if mode == "rr" else kd.build_widest_cuda)(d)
    # and the next clean build succeeds (the flag is per build)
    p = datagen.uniform(n, 3, seed=n + 1)
    _, perm = kd.build_round_robin_cuda(_dev(p))
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.rec_build(p))


def test_caller_buffers_are_validated():
    """wrong dtype / shape / device of out, perm,
    split_dims raise instead of letting the native code write past them."""
    d = _dev(datagen.uniform(1000, 3, seed=1))
    with pytest.raises(ValueError):
        kd.build_round_robin_cuda(d, out=torch.empty((999, 3), device="cuda"))
    with pytest.raises(ValueError):
        kd.build_round_robin_cuda(d, out=torch.empty((1000, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        kd.build_round_robin_cuda(d, perm=torch.empty(999, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        kd.build_round_robin_cuda(d, perm=torch.empty(1000, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError):
        kd.build_widest_cuda(d, split_dims=torch.empty(1000, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        kd.build_round_robin_cuda(d, out=torch.empty((1000, 3)))
    with pytest.raises(ValueError):
        kd.build_round_robin_cuda(d.to(torch.int32))
    with pytest.raises(ValueError):  # float64 points need float64 out
        kd.build_round_robin_cuda(d.double(), out=torch.empty((1000, 3), device="cuda"))


def test_query_cache_sees_in_place_edits():
    """the device copy of a tree used by check_valid /
    knn must follow in-place edits of tree.coords and tree.split_dims."""
    from paper_2211_00120_b200 import verify

    pts = datagen.uniform(5000, 3, seed=4)
    tree = kd.build_round_robin(pts)
    assert verify.check_valid(tree).valid
    nb = kd.knn(tree, pts[17].astype(np.float64), 1)
    assert nb[0].dist2 == 0.0
    # nudge a leaf inside its own cell: a stale device copy would report the
    # old position (dist2 > 0), a fresh one finds the leaf exactly
    leaf = tree.n - 1
    tree.coords[leaf] = np.nextafter(tree.coords[leaf], np.inf)
    nb = kd.knn(tree, tree.coords[leaf].copy(), 1)
    assert nb[0].index == leaf and nb[0].dist2 == 0.0
    # move node 1 (left child of the root) to the far right of the root plane
    tree.coords[1, 0] = tree.coords[0, 0] + 10.0
    assert not verify.check_valid(tree).valid
    wt = kd.build_widest(pts)
    assert verify.check_valid(wt).valid
    s = int(np.argmax(wt.split_dims[:7] != 0))
    wt.split_dims[s] = (wt.split_dims[s] + 1) % 3
    rep = verify.check_valid(wt)
    wt.split_dims[s] = (wt.split_dims[s] + 2) % 3
    assert verify.check_valid(wt).valid
    del rep
