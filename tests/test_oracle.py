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
    return [v for v in h.values() if v["n"] <= 1_000_000]


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
