"""GPU kNN / radius queries (csrc/query.cu) against the reference's answers
(golden/queries.npz) and the oracle's brute-force scans -- exact: same
indices, bit-identical float64 squared distances.  Mirrors the reference's
tests/test_queries.py (knn vs scan, ordering, exact ties by index,
duplicates, radius vs scan, boundary included, zero radius)."""

import numpy as np
import pytest

from oracle import oracle
from tests.golden_util import gen_case, query_cases

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import build_round_robin, build_widest, datagen, queries  # noqa: E402


def build_any(rng, coords, k):
    if rng.integers(2):
        return build_widest(coords, k)
    return build_round_robin(coords, k)


def test_golden_reference_answers():
    for case in query_cases():
        pts = gen_case(case)
        tree = (build_round_robin if case["mode"] == "rr" else build_widest)(pts, case["k"])
        assert np.array_equal(tree.payload, case["payload"]), case["name"]
        for qi, q in enumerate(case["queries"]):
            for m, want in case["knn"][qi].items():
                got = [(nb.index, nb.dist2) for nb in queries.knn(tree, q, m)]
                assert got == want, (case["name"], qi, m)
            for r, want in zip(case["radii"], case["radius"][qi]):
                assert np.array_equal(queries.radius_query(tree, q, r), want), (case["name"], qi, r)


def test_golden_batched_matches_single():
    for case in query_cases()[::4]:
        pts = gen_case(case)
        tree = (build_round_robin if case["mode"] == "rr" else build_widest)(pts, case["k"])
        for m in (1, 17):
            idx, d2 = queries.knn_batch(tree, case["queries"], m)
            for qi in range(len(case["queries"])):
                assert list(zip(idx[qi].tolist(), d2[qi].tolist())) == case["knn"][qi][m], (case["name"], m)
        off, hits = queries.radius_batch(tree, case["queries"], case["radii"][2])
        for qi in range(len(case["queries"])):
            assert np.array_equal(hits[off[qi]:off[qi + 1]], case["radius"][qi][2])


def test_knn_matches_scan():
    rng = np.random.default_rng(211)
    for _ in range(40):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, 5))
        coords = (rng.random((n, k)) * 10).astype(np.float32)
        tree = build_any(rng, coords, k)
        query = rng.random(k) * 12 - 1
        for m in (1, 5, 17, 33, n + 3):
            got = [tuple(nb) for nb in queries.knn(tree, query, m)]
            assert got == oracle.brute_knn(tree.coords, query, m), (n, k, m)


def test_knn_exact_ties_break_by_index():
    coords = np.array([[1.0, 0.0], [-1.0, 0.0], [0.0, 1.0], [0.0, -1.0], [5.0, 5.0]], dtype=np.float32)
    for build in (build_round_robin, build_widest):
        tree = build(coords, 2)
        got = queries.knn(tree, [0.0, 0.0], 3)
        assert [nb.dist2 for nb in got] == [1.0, 1.0, 1.0]
        tied = np.flatnonzero((tree.coords ** 2).sum(axis=1) == 1.0)
        assert [nb.index for nb in got] == tied.tolist()[:3]


def test_knn_with_duplicate_points():
    rng = np.random.default_rng(227)
    for _ in range(25):
        n = int(rng.integers(1, 200))
        k = int(rng.integers(1, 4))
        coords = rng.integers(0, 3, size=(n, k)).astype(np.float32)
        tree = build_any(rng, coords, k)
        query = rng.integers(0, 3, size=k).astype(np.float64)
        for m in (1, 4, 17, 64):
            got = [tuple(nb) for nb in queries.knn(tree, query, m)]
            assert got == oracle.brute_knn(tree.coords, query, m)


def test_radius_matches_scan_boundary_and_zero():
    rng = np.random.default_rng(233)
    for _ in range(40):
        n = int(rng.integers(1, 300))
        k = int(rng.integers(1, 5))
        coords = (rng.random((n, k)) * 4).astype(np.float32)
        tree = build_any(rng, coords, k)
        query = rng.random(k) * 4
        for radius in (0.0, float(rng.random()), 2.5, 10.0):
            got = queries.radius_query(tree, query, radius)
            assert np.array_equal(got, oracle.brute_radius(tree.coords, query, radius)), (n, k, radius)
    coords = np.array([[0.0, 0.0], [3.0, 0.0], [0.0, 4.0], [6.0, 6.0]], dtype=np.float32)
    tree = build_round_robin(coords, 2)
    assert {tuple(tree.coords[i]) for i in queries.radius_query(tree, [0.0, 0.0], 3.0)} == {(0.0, 0.0), (3.0, 0.0)}
    coords = np.array([[1.0, 1.0], [1.0, 1.0], [2.0, 2.0]], dtype=np.float32)
    tree = build_round_robin(coords, 2)
    got = queries.radius_query(tree, [1.0, 1.0], 0.0)
    assert len(got) == 2 and all(tuple(tree.coords[i]) == (1.0, 1.0) for i in got)


def test_errors_match_reference():
    tree = build_round_robin(np.zeros((0, 2), dtype=np.float32), 2)
    with pytest.raises(ValueError, match="empty tree"):
        queries.knn(tree, [0.0, 0.0], 1)
    assert queries.radius_query(tree, [0.0, 0.0], 1.0).shape == (0,)
    tree = build_round_robin(np.random.default_rng(1).random((10, 2)).astype(np.float32), 2)
    with pytest.raises(ValueError, match="at least 1"):
        queries.knn(tree, [0.0, 0.0], 0)
    with pytest.raises(ValueError, match="dimensions"):
        queries.knn(tree, [0.0, 0.0, 0.0], 1)
    with pytest.raises(ValueError, match="finite"):
        queries.knn(tree, [np.nan, 0.0], 1)
    with pytest.raises(ValueError, match="non-negative"):
        queries.radius_query(tree, [0.0, 0.0], -1.0)


@pytest.mark.parametrize("mode", ["rr", "widest"])
def test_large_batch_on_device_tree(mode):
    """1M-point tree straight from the device build, 4096 queries; a sample
    of them checked against full scans (kNN m = 8 and 48 -- the local and the
    global keep-list kernels -- and radius, one query with > 4096 hits so the
    global-memory sort runs)."""
    n, k = 1_000_000, 3
    pts = datagen.make("clustered" if mode == "widest" else "uniform", n, k, seed=5)
    d = torch.from_numpy(pts).cuda()
    if mode == "rr":
        out, perm = kd.build_round_robin_cuda(d)
        dims = None
    else:
        out, perm, dims = kd.build_widest_cuda(d)
    host = out.cpu().numpy().astype(np.float64)
    rng = np.random.default_rng(9)
    qn = rng.random((4096, k))
    qn[:64] = host[rng.integers(0, n, 64)]
    q = torch.from_numpy(qn).cuda()
    sample = list(range(0, 64, 8)) + list(range(64, 4096, 509))
    for m in (8, 48):
        idx, d2 = queries.knn_cuda(out, q, m, split_dims=dims)
        idx, d2 = idx.cpu().numpy(), d2.cpu().numpy()
        for qi in sample:
            want = oracle.brute_knn(host, qn[qi], m)
            assert list(zip(idx[qi].tolist(), d2[qi].tolist())) == want, (mode, m, qi)
    qb = qn.copy()
    qb[0] = [0.5, 0.5, 0.5]
    q = torch.from_numpy(qb).cuda()
    off, hits = queries.radius_cuda(out, q, 0.12, split_dims=dims)
    off, hits = off.cpu().numpy(), hits.cpu().numpy()
    assert off[1] - off[0] > 4096
    for qi in [0] + sample:
        assert np.array_equal(hits[off[qi]:off[qi + 1]], oracle.brute_radius(host, qb[qi], 0.12)), (mode, qi)
