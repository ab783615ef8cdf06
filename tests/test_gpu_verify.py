"""GPU check_valid / brute_subtree_boxes (csrc/verify.cu) against the oracle
restatements of verify.check_valid (+ its witness) and
verify.brute_subtree_boxes; exact."""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import build_round_robin, build_widest, datagen, verify  # noqa: E402


def trees():
    rng = np.random.default_rng(7)
    for kind in ("uniform", "clustered", "ties"):
        for k in (1, 2, 3, 4):
            n = int(rng.integers(2, 3000))
            pts = datagen.make(kind, n, k, seed=int(rng.integers(1 << 30)))
            yield f"rr-{kind}-{n}-{k}", build_round_robin(pts, k)
            yield f"widest-{kind}-{n}-{k}", build_widest(pts, k)


def test_built_trees_are_valid_and_boxes_match():
    for name, tree in trees():
        rep = verify.check_valid(tree)
        assert rep.valid and oracle.check_valid(tree.coords, tree.split_dims), name
        lo, hi = verify.brute_subtree_boxes(tree)
        wlo, whi = oracle.brute_subtree_boxes(tree.coords, tree.split_dims)
        assert np.array_equal(lo, wlo) and np.array_equal(hi, whi), name


def test_planted_violations_give_the_reference_witness():
    rng = np.random.default_rng(11)
    hits = 0
    for name, tree in trees():
        for _ in range(3):
            bad = kd.KdTree(tree.coords.copy(), tree.payload, tree.split_dims)
            i, j = rng.integers(0, tree.n, 2)
            bad.coords[[i, j]] = bad.coords[[j, i]]
            want = oracle.validity_witness(bad.coords, bad.split_dims)
            rep = verify.check_valid(bad)
            if want is None:
                assert rep.valid, name
                continue
            hits += 1
            assert not rep.valid and (rep.descendant, rep.ancestor, rep.dim) == want, name
            assert f"node {want[0]} (" in rep.message and f"subtree of node {want[1]}" in rep.message
    assert hits > 10


def test_device_tree_100k():
    n, k = 100_000, 3
    pts = datagen.make("uniform", n, k, seed=3)
    out, perm, dims = kd.build_widest_cuda(torch.from_numpy(pts).cuda())
    assert verify.check_valid_cuda(out, split_dims=dims) is None
    lo, hi = verify.subtree_boxes_cuda(out, split_dims=dims)
    host = out.cpu().numpy()
    wlo, whi = oracle.brute_subtree_boxes(host, dims.cpu().numpy())
    assert np.array_equal(lo.cpu().numpy(), wlo) and np.array_equal(hi.cpu().numpy(), whi)
    # one corrupted coordinate deep in the tree is found
    out[n - 1, :] = 1e9  # node n-1 lies in the left subtree of some ancestor
    w = verify.check_valid_cuda(out, split_dims=dims)
    assert w is not None and w == oracle.validity_witness(out.cpu().numpy(), dims.cpu().numpy())
