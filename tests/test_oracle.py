"""Pin the CPU oracle against the reference's own outputs (CPU only).

The golden vectors in tests/golden/ were produced by running the reference
package (tests/golden/make_golden.py); this file checks that the C
restatement in oracle/ reproduces them bit for bit, so the GPU parity tests
can trust it as the checker.
"""

import json
import os
import hashlib

import numpy as np
import pytest

from oracle import oracle
from tests.golden_util import GOLDEN, gen_case, query_cases, small_cases


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_walkthrough_every_phase():
    g = np.load(os.path.join(GOLDEN, "walkthrough.npz"))
    pts = g["points"]
    perm, tags, idx = oracle.build_rr(pts, trace=True)
    assert tags.shape == g["tags"].shape
    for ph in range(tags.shape[0]):
        assert tags[ph].tolist() == g["tags"][ph].tolist(), ph
        assert np.array_equal(pts[idx[ph]], g["coords"][ph]), ph
    assert perm.tolist() == g["perm"].tolist()
    # final x/y rows of the reference walkthrough (test_acceptance.py:26-28)
    assert pts[perm, 0].tolist() == [46, 15, 53, 40, 44, 68, 62, 10, 45, 25]
    assert pts[perm, 1].tolist() == [63, 43, 67, 33, 58, 21, 69, 15, 40, 54]


def test_small_cases_bit_exact():
    for case in small_cases():
        pts = gen_case(case)
        if case["mode"] == "rr":
            perm = oracle.build_rr(pts)
            assert np.array_equal(perm, case["perm"]), case["name"]
        else:
            perm, dims = oracle.build_widest(pts)
            assert np.array_equal(perm, case["perm"]), case["name"]
            assert np.array_equal(dims, case["split_dims"]), case["name"]


def _medium():
    h = json.load(open(os.path.join(GOLDEN, "hashes.json")))
    return [v for v in h.values() if v["n"] <= 1_000_000 and v.get("source", "reference") == "reference"]


@pytest.mark.parametrize("case", _medium(), ids=lambda c: f"{c['mode']}-{c['kind']}-{c['n']}-k{c['k']}")
def test_medium_hashes(case):
    pts = gen_case(case)
    assert sha(pts) == case["input_sha256"], "input generator drifted"
    if case["mode"] == "rr":
        perm = oracle.build_rr(pts)
    else:
        perm, dims = oracle.build_widest(pts)
        assert sha(dims) == case["split_dims_sha256"]
    assert perm[:64].tolist() == case["perm_head"]
    assert sha(perm) == case["perm_sha256"]


def test_check_valid_and_boxes_on_oracle_trees():
    rng = np.random.default_rng(3)
    for _ in range(20):
        n = int(rng.integers(1, 400))
        k = int(rng.integers(1, 5))
        pts = rng.integers(0, 3, size=(n, k)).astype(np.float32)
        perm = oracle.build_rr(pts)
        assert oracle.check_valid(pts[perm])
        perm, dims = oracle.build_widest(pts)
        assert oracle.check_valid(pts[perm], dims)
        lo, hi = oracle.brute_subtree_boxes(pts[perm], dims)
        assert np.array_equal(dims.astype(np.int64), np.argmax(hi - lo, axis=1))


def test_check_valid_catches_planted_violation():
    pts = np.random.default_rng(313).random((63, 2)).astype(np.float32)
    perm = oracle.build_rr(pts)
    tree = pts[perm].copy()
    tree[40, 0] = tree[0, 0] + 100.0
    assert not oracle.check_valid(tree)


def test_query_checkers_match_reference_answers():
    """oracle.brute_knn / brute_radius against the reference's own
    queries.knn / radius_query answers (golden/queries.npz)."""
    for case in query_cases():
        pts = gen_case(case)
        coords = pts[case["payload"]].astype(np.float64)  # the reference tree
        for qi, q in enumerate(case["queries"]):
            for m, want in case["knn"][qi].items():
                assert oracle.brute_knn(coords, q, m) == want, (case["name"], qi, m)
            for r, want in zip(case["radii"], case["radius"][qi]):
                assert np.array_equal(oracle.brute_radius(coords, q, r), want), (case["name"], qi, r)


# --- the recursive oracle (oracle/lbkd_recursive.cpp, verify.py:121-168) ----

def test_recursive_oracle_small_golden_cases():
    """The threaded recursive restatement reproduces every reference-run
    small case (RR and widest, ties, +-0.0, clustered negatives)."""
    for case in small_cases():
        pts = gen_case(case)
        if case["mode"] == "rr":
            assert np.array_equal(oracle.rec_build(pts), case["perm"]), case["name"]
        else:
            perm, dims = oracle.rec_build(pts, widest=True)
            assert np.array_equal(perm, case["perm"]), case["name"]
            assert np.array_equal(dims, case["split_dims"]), case["name"]


@pytest.mark.parametrize("case", _medium(), ids=lambda c: f"{c['mode']}-{c['kind']}-{c['n']}-k{c['k']}")
def test_recursive_oracle_medium_hashes(case):
    pts = gen_case(case)
    if case["mode"] == "rr":
        perm = oracle.rec_build(pts, threads=4)
    else:
        perm, dims = oracle.rec_build(pts, widest=True, threads=4)
        assert sha(dims) == case["split_dims_sha256"]
    assert sha(perm) == case["perm_sha256"]


def test_recursive_oracle_equals_tag_and_sort_under_ties():
    """SURVEY.md Appendix A.7 as a test: the recursive oracle and the
    tag-and-sort restatement agree on tie-heavy inputs, both modes, and the
    thread count does not change the result."""
    rng = np.random.default_rng(17)
    for t in range(40):
        n = int(rng.integers(2, 5000))
        k = int(rng.integers(1, 5))
        q = [2, 3, 8, 64, 0][t % 5]
        pts = rng.random((n, k), dtype=np.float32)
        if q:
            pts = (np.floor(pts * q) / q).astype(np.float32)
        a = oracle.build_rr(pts)
        assert np.array_equal(oracle.rec_build(pts, threads=1), a), (t, n, k, q)
        assert np.array_equal(oracle.rec_build(pts, threads=8), a), (t, n, k, q)
        wp, wd = oracle.build_widest(pts)
        rp, rd = oracle.rec_build(pts, widest=True, threads=3)
        assert np.array_equal(rp, wp) and np.array_equal(rd, wd), (t, n, k, q)


def test_recursive_oracle_float64_matches_float32_promotion():
    """float64 input that is exactly float32-representable gives the same
    tree through the float64 instantiation (the reference promotes)."""
    pts = (np.floor(np.random.default_rng(5).random((30000, 3)) * 50) / 50).astype(np.float32)
    assert np.array_equal(oracle.rec_build(pts.astype(np.float64)), oracle.rec_build(pts))
    a = oracle.rec_build(pts.astype(np.float64), widest=True)
    b = oracle.rec_build(pts, widest=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_recursive_oracle_float64_reference_hashes():
    """The float64 instantiation of the recursive oracle reproduces the
    reference's own outputs on float64 inputs that are not float32-exact
    (tests/golden/hashes_f64.json, made by running the reference)."""
    from tests.golden_util import f64_cases, gen_f64

    for c in f64_cases():
        pts = gen_f64(c["kind"], c["n"], c["k"], c["seed"])
        assert sha(pts) == c["input_sha256"], "input generator drifted"
        if c["mode"] == "rr":
            perm = oracle.rec_build(pts, threads=4)
        else:
            perm, dims = oracle.rec_build(pts, widest=True, threads=4)
            assert sha(dims) == c["split_dims_sha256"], c
        assert sha(perm) == c["perm_sha256"], c
        assert sha(pts[perm.astype(np.int64)]) == c["coords_sha256"], c
