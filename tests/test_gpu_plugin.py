"""The reference's kernel-plugin seam with this repo's module
(paper_2211_00120_b200.kernels_b200): the UNMODIFIED reference loop
(baseline/_ref: its own lexsort, its own driver) calls our
lbkd_update_tags_rr / lbkd_update_tags_widest / lbkd_knn_f64 /
lbkd_radius_*_f64 through accel.get_kernels() (accel.py:48-58), and every
result must equal the reference's own numpy backend."""

import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "lbkd")):
    pytest.skip("baseline/_ref (the reference install) is absent", allow_module_level=True)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/lbkd_plugin_numba")
sys.path.insert(0, REF)

import lbkd  # noqa: E402  (the reference)
import lbkd.builder  # noqa: E402
import lbkd.queries  # noqa: E402
import lbkd.widest  # noqa: E402

from paper_2211_00120_b200 import kernels_b200  # noqa: E402


@pytest.fixture
def plugin(monkeypatch):
    """accel.get_kernels() -> kernels_b200 in every reference module."""
    for mod in (lbkd.builder, lbkd.widest, lbkd.queries):
        monkeypatch.setattr(mod, "get_kernels", lambda: kernels_b200)
    yield
    # (monkeypatch restores the reference dispatch)


def _inputs():
    rng = np.random.default_rng(23)
    yield rng.random((3000, 3))
    yield (np.floor(rng.random((5000, 2)) * 16) / 16)
    yield rng.choice(np.array([0.0, -0.0, 1.0, -1.0]), size=(2000, 3))
    yield rng.random((40000, 4)) * np.array([1.0, 10.0, 0.1, 3.0])
    c = rng.random((64, 3))
    yield c[rng.integers(0, 64, 20000)] + rng.normal(0, 0.01, (20000, 3))


def _ref(fn, pts, monkeypatch_env):
    monkeypatch_env.setenv("LBKD_BACKEND", "numpy")
    return fn(pts, pts.shape[1])


def test_update_kernels_through_the_plugin_seam(plugin, monkeypatch):
    for pts in _inputs():
        for fn in (lbkd.builder.build_round_robin, lbkd.widest.build_widest):
            got = fn(pts, pts.shape[1])  # the reference loop, our update kernels
            monkeypatch.setattr(lbkd.builder, "get_kernels", lbkd.accel.get_kernels)
            monkeypatch.setattr(lbkd.widest, "get_kernels", lbkd.accel.get_kernels)
            want = _ref(fn, pts, monkeypatch)
            monkeypatch.setattr(lbkd.builder, "get_kernels", lambda: kernels_b200)
            monkeypatch.setattr(lbkd.widest, "get_kernels", lambda: kernels_b200)
            assert np.array_equal(got.payload, want.payload), (fn.__name__, pts.shape)
            assert np.array_equal(got.coords, want.coords)
            if want.split_dims is not None:
                assert np.array_equal(got.split_dims, want.split_dims), (fn.__name__, pts.shape)


def test_query_kernels_through_the_plugin_seam(plugin, monkeypatch):
    rng = np.random.default_rng(5)
    for pts in _inputs():
        monkeypatch.setenv("LBKD_BACKEND", "numpy")
        for build in (lbkd.builder.build_round_robin, lbkd.widest.build_widest):
            monkeypatch.setattr(lbkd.builder, "get_kernels", lbkd.accel.get_kernels)
            monkeypatch.setattr(lbkd.widest, "get_kernels", lbkd.accel.get_kernels)
            tree = build(pts, pts.shape[1])
            for _ in range(6):
                q = pts[rng.integers(0, len(pts))] + rng.normal(0, 0.05, pts.shape[1])
                monkeypatch.setattr(lbkd.queries, "get_kernels", lbkd.accel.get_kernels)
                want_knn = lbkd.queries.knn(tree, q, 7)
                want_rad = lbkd.queries.radius_query(tree, q, 0.2)
                monkeypatch.setattr(lbkd.queries, "get_kernels", lambda: kernels_b200)
                assert lbkd.queries.knn(tree, q, 7) == want_knn
                assert np.array_equal(lbkd.queries.radius_query(tree, q, 0.2), want_rad)
