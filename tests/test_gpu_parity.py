"""GPU parity: the CUDA build against the reference's golden vectors and the
CPU oracle (oracle/), bit-exact, through the public API and the C-ABI."""

import hashlib
import json
import os

import numpy as np
import pytest

from oracle import oracle
from tests.golden_util import GOLDEN, gen_case, small_cases

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import BuildRecorder, build_round_robin, build_widest  # noqa: E402
from paper_2211_00120_b200 import datagen  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def gpu_rr(pts):
    d = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32)).cuda()
    out, perm = kd.build_round_robin_cuda(d)
    return out.cpu().numpy(), perm.cpu().numpy().view(np.uint32)


def gpu_widest(pts):
    d = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32)).cuda()
    out, perm, dims = kd.build_widest_cuda(d)
    return out.cpu().numpy(), perm.cpu().numpy().view(np.uint32), dims.cpu().numpy()


def test_walkthrough_every_phase():
    g = np.load(os.path.join(GOLDEN, "walkthrough.npz"))
    rec = BuildRecorder(capture=True)
    tree = build_round_robin(g["points"], recorder=rec)
    assert len(rec.snapshots) == g["tags"].shape[0]
    for i, snap in enumerate(rec.snapshots):
        assert snap.event == str(g["events"][i])
        assert snap.iteration == int(g["iterations"][i])
        assert snap.tags.tolist() == g["tags"][i].tolist(), i
        assert np.array_equal(snap.coords, g["coords"][i].astype(np.float64)), i
    assert tree.coords[:, 0].tolist() == [46, 15, 53, 40, 44, 68, 62, 10, 45, 25]
    assert tree.coords[:, 1].tolist() == [63, 43, 67, 33, 58, 21, 69, 15, 40, 54]
    assert rec.sort_phases == 4 and rec.update_phases == 3 and rec.tag_bytes == 40


def test_small_golden_cases_bit_exact():
    for case in small_cases():
        pts = gen_case(case)
        if case["mode"] == "rr":
            out, perm = gpu_rr(pts)
            assert np.array_equal(perm, case["perm"]), case["name"]
        else:
            out, perm, dims = gpu_widest(pts)
            assert np.array_equal(perm, case["perm"]), case["name"]
            assert np.array_equal(dims, case["split_dims"]), case["name"]
        assert np.array_equal(out, pts[case["perm"].astype(np.int64)]), case["name"]


def _hash_cases(max_n):
    h = json.load(open(os.path.join(GOLDEN, "hashes.json")))
    # reference-generated entries (the 1B entry comes from the recursive
    # oracle and has its own test, tests/test_gpu_big.py)
    return [v for v in h.values() if v["n"] <= max_n and v.get("source", "reference") == "reference"]


@pytest.mark.parametrize("case", _hash_cases(10**9), ids=lambda c: f"{c['mode']}-{c['kind']}-{c['n']}-k{c['k']}")
def test_golden_hashes(case):
    pts = gen_case(case)
    assert sha(pts) == case["input_sha256"]
    if case["mode"] == "rr":
        out, perm = gpu_rr(pts)
    else:
        out, perm, dims = gpu_widest(pts)
        assert sha(dims) == case["split_dims_sha256"]
    assert perm[:64].tolist() == case["perm_head"]
    assert sha(perm) == case["perm_sha256"]
    # the reordered points are the input rows in node order
    step = max(1, len(perm) // 100000)
    assert np.array_equal(out[::step], pts[perm[::step].astype(np.int64)])


SIZES = [1, 2, 3, 7, 8, 100, 4095, 8191, 8192, 8193, 12287, 16383, 16384, 16385, 40000, 65535, 65536, 65537,
         131071, 200003, 262144, 300001, 524287, 1 << 20]


@pytest.mark.parametrize("n", SIZES)
def test_rr_vs_oracle_sizes(n):
    rng = np.random.default_rng(n)
    for kind in ("uniform", "ties", "clustered", "signed_zero"):
        k = int(rng.integers(1, 6))
        pts = datagen.make(kind, n, k, seed=n + k)
        _, perm = gpu_rr(pts)
        assert np.array_equal(perm, oracle.build_rr(pts)), (kind, n, k)


@pytest.mark.parametrize("n", SIZES)
def test_widest_vs_oracle_sizes(n):
    rng = np.random.default_rng(n + 1)
    for kind in ("uniform", "ties", "clustered"):
        k = int(rng.integers(1, 6))
        pts = datagen.make(kind, n, k, seed=n + 2 * k)
        _, perm, dims = gpu_widest(pts)
        want_perm, want_dims = oracle.build_widest(pts)
        assert np.array_equal(perm, want_perm), (kind, n, k)
        assert np.array_equal(dims, want_dims), (kind, n, k)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 8, 12, 16])
def test_all_dimension_counts(k):
    for n in (5000, 70001):
        pts = datagen.ties(n, k, seed=k)
        _, perm = gpu_rr(pts)
        assert np.array_equal(perm, oracle.build_rr(pts)), (n, k)
        _, perm, dims = gpu_widest(pts)
        wp, wd = oracle.build_widest(pts)
        assert np.array_equal(perm, wp), (n, k)
        assert np.array_equal(dims, wd), (n, k)


def test_in_place_and_payload():
    pts = datagen.uniform(50000, 3, seed=9)
    d = torch.from_numpy(pts).cuda()
    ref = oracle.build_rr(pts)
    out, perm = kd.build_round_robin_cuda(d, out=d)  # in place
    assert out.data_ptr() == d.data_ptr()
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), ref)
    assert np.array_equal(d.cpu().numpy(), pts[ref.astype(np.int64)])
    payload = np.arange(50000, dtype=np.int64) * 7 + 3
    tree = build_round_robin(pts, 3, payload=payload)
    assert np.array_equal(tree.payload, payload[ref.astype(np.int64)])
    assert tree.coords.dtype == np.float64


def test_edge_cases_and_validation():
    empty = build_round_robin(np.empty((0, 2), dtype=np.float32), 2)
    assert empty.n == 0 and empty.k == 2 and empty.levels == 0
    one = build_round_robin(np.array([[3.5, 2.5]], dtype=np.float32), 2)
    assert one.coords.tolist() == [[3.5, 2.5]] and one.payload.tolist() == [0]
    t = build_round_robin([5.0, 1.0, 9.0])
    assert t.coords[:, 0].tolist() == [5.0, 1.0, 9.0]
    w = build_widest(np.array([[2.0, 9.0]], dtype=np.float32), 2)
    assert w.split_dims.tolist() == [0]
    ew = build_widest(np.empty((0, 4), dtype=np.float32), 4)
    assert ew.split_dims.shape == (0,)
    same = build_round_robin(np.full((25, 3), 4.25, dtype=np.float32), 3)
    assert sorted(same.payload.tolist()) == list(range(25))
    # reference hand cases (tests/test_verify.py:9-25)
    assert build_round_robin([[5.0], [1.0]]).coords[:, 0].tolist() == [5.0, 1.0]
    assert build_round_robin([[3.0], [1.0], [7.0], [5.0]]).coords[:, 0].tolist() == [5.0, 3.0, 7.0, 1.0]
    with pytest.raises(ValueError):
        build_round_robin(np.array([[1.0], [np.nan]], dtype=np.float32))
    # the device flag catches non-finite input that skips host validation
    bad = torch.tensor([[1.0, 2.0], [float("inf"), 0.0]] * 5000, device="cuda")
    with pytest.raises(ValueError, match="finite"):
        kd.build_round_robin_cuda(bad)
    with pytest.raises(ValueError):
        build_widest(np.broadcast_to(np.zeros((1, 3), dtype=np.float32), (2**29, 3)))


def test_recorder_counts():
    for n in (1, 2, 3, 10, 100, 1000, 20000):
        rec = BuildRecorder()
        build_round_robin(datagen.uniform(n, 2, seed=n), 2, recorder=rec)
        L = n.bit_length()
        assert (rec.sort_phases, rec.update_phases, rec.tag_entries, rec.tag_itemsize) == (L, L - 1, n, 4)


def test_widest_recorder_capture_matches_oracle_dims():
    pts = datagen.uniform(300, 3, seed=4)
    rec = BuildRecorder(capture=True)
    tree = build_widest(pts, 3, recorder=rec)
    wp, wd = oracle.build_widest(pts)
    assert np.array_equal(tree.payload, wp.astype(np.int64))
    assert np.array_equal(tree.split_dims, wd)
    assert len(rec.snapshots) == 2 * (300).bit_length()


def test_plugin_seam_update_kernels_match_oracle_trace():
    from paper_2211_00120_b200 import _native

    lib = _native.load()
    pts = datagen.ties(3000, 3, seed=1)
    perm, tags, idx = oracle.build_rr(pts, trace=True)
    n = 3000
    L = n.bit_length()
    for l in range(L - 1):
        before = tags[1 + 2 * l]  # after sort l
        after = tags[2 + 2 * l]   # after update l
        d = torch.from_numpy(before.view(np.int32).copy()).cuda()
        rc = lib.lbkd_update_tags_rr(d.data_ptr(), n, L, l, None)
        assert rc == 0
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy().view(np.uint32), after), l


def test_check_valid_at_scale():
    for kind in ("uniform", "clustered"):
        pts = datagen.make(kind, 4_000_000, 3, seed=11)
        out, perm = gpu_rr(pts)
        assert np.array_equal(np.sort(perm), np.arange(len(perm), dtype=np.uint32))
        assert oracle.check_valid(out)
        out, perm, dims = gpu_widest(pts)
        assert oracle.check_valid(out, dims)


@pytest.mark.parametrize("n,k,world,kind", [(300_000, 3, 2, "uniform"), (1_000_000, 3, 8, "clustered"),
                                            (2_000_003, 2, 4, "ties"), (500_000, 4, 4, "uniform"),
                                            (20_000, 3, 4, "uniform"), (70_000, 1, 2, "ties")])
def test_sharded_build_matches_single_gpu(n, k, world, kind):
    """The multi-GPU path run rank by rank on one GPU: top levels, then every
    subtree from its packed points with the global geometry -- bit-identical
    to the single-device build (the exchange itself is covered by the gloo
    tests)."""
    from paper_2211_00120_b200 import multigpu

    pts = datagen.make(kind, n, k, seed=n)
    d = torch.from_numpy(pts).cuda()
    want_out, want_perm = kd.build_round_robin_cuda(d)
    top = multigpu.top_levels_for(world)
    ops = multigpu.CudaOps(0)
    out = torch.full_like(d, float("nan"))
    perm = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    sub = torch.empty((k + 1) * n, dtype=torch.int32, device="cuda")
    ops.build_top(d, top, out, perm, sub, n)
    for sh in multigpu.shard_layout(n, top):
        mine = torch.empty((k + 1) * sh.size, dtype=torch.int32, device="cuda")
        for c in range(k + 1):
            mine[c * sh.size:(c + 1) * sh.size] = sub[c * n + sh.offset: c * n + sh.offset + sh.size]
        ops.build_sub(mine, sh.size, n, k, top, sh.index, out, perm)
    torch.cuda.synchronize()
    assert torch.equal(perm, want_perm)
    assert torch.equal(out, want_out)
    assert oracle.build_rr(pts).tolist()[:1000] == perm.cpu().numpy().view(np.uint32).tolist()[:1000]
    # the recursive-halving protocol (lbkd_build_rr_top with one level, then
    # lbkd_build_rr_split per step, then lbkd_build_rr_sub) run rank by rank
    out2, perm2 = multigpu.serial_sharded_build(d, n, k, world)
    torch.cuda.synchronize()
    assert torch.equal(perm2, want_perm)
    assert torch.equal(out2, want_out)


@pytest.mark.parametrize("n", [8193, 70001, 300001, 1 << 20])
def test_sort_algorithm_matches_oracle(n):
    """The literal per-level radix-sort path (LBKD_ALGO=sort: onesweep digit
    passes over every segment) is bit-exact too."""
    from paper_2211_00120_b200 import _native

    _native.set_algorithm("sort")
    try:
        assert _native.get_algorithm() == "sort"
        for kind, k in (("uniform", 3), ("ties", 2), ("clustered", 4)):
            pts = datagen.make(kind, n, k, seed=n + k)
            _, perm = gpu_rr(pts)
            assert np.array_equal(perm, oracle.build_rr(pts)), (kind, n, k)
            _, perm, dims = gpu_widest(pts)
            wp, wd = oracle.build_widest(pts)
            assert np.array_equal(perm, wp) and np.array_equal(dims, wd), (kind, n, k)
    finally:
        _native.set_algorithm("select")


def test_profile_classes_cover_the_build():
    """lbkd_profile_kernel accounts every kernel of a profiled build."""
    from paper_2211_00120_b200 import _native

    pts = datagen.uniform(1 << 20, 3, seed=5)
    d = torch.from_numpy(pts).cuda()
    kd.build_round_robin_cuda(d)
    _native.set_profile(True)
    try:
        kd.build_round_robin_cuda(d)
        torch.cuda.synchronize()
        prof = _native.profile_kernels()
    finally:
        _native.set_profile(False)
    assert {"init", "hist", "pick", "filter", "select", "partition", "subtree"} <= set(prof)
    n_launch = sum(v[0] for v in prof.values())
    assert n_launch == kd.builder.last_launch_count(0)
    part = prof["partition"]
    assert part[1] > 0 and part[2] > 0


@pytest.mark.parametrize("algo", ["sort", "select"])
def test_profiled_ungraphed_builds(algo):
    """Profiling an ungraphed build (the sort path; float64 widest, whose
    value table is a kernel argument) records plain events and stays exact."""
    from paper_2211_00120_b200 import _native

    pts = datagen.uniform(300001, 3, seed=7)
    ref = oracle.build_rr(pts)
    _native.set_algorithm(algo)
    _native.set_profile(True)
    try:
        _, perm = gpu_rr(pts)
        assert np.array_equal(perm, ref)
        assert sum(v[0] for v in _native.profile_kernels().values()) == kd.builder.last_launch_count(0)
        p64 = np.random.default_rng(3).random((50001, 3))
        t = build_widest(p64)
        wp, wd = oracle.rec_build(p64, widest=True)
        assert np.array_equal(t.payload, wp.astype(np.int64)) and np.array_equal(t.split_dims, wd)
    finally:
        _native.set_profile(False)
        _native.set_algorithm("select")


def test_pipelined_host_builds():
    """lbkd_build_rr_host: consecutive host-buffer builds overlap and each
    returns its own exact result; a non-finite input is reported at join."""
    from paper_2211_00120_b200.builder import build_round_robin_host, host_join

    n, k = 300001, 3
    inputs = [datagen.make(kind, n, k, seed=s) for s, kind in enumerate(("uniform", "ties", "clustered"))]
    hin = [torch.from_numpy(p).pin_memory() for p in inputs]
    hout = [torch.empty((n, k), dtype=torch.float32).pin_memory() for _ in inputs]
    hperm = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in inputs]
    for i in range(len(inputs)):
        build_round_robin_host(hin[i], hout[i], hperm[i])
    host_join()
    for i, p in enumerate(inputs):
        want = oracle.build_rr(p)
        assert np.array_equal(hperm[i].numpy().view(np.uint32), want), i
        assert np.array_equal(hout[i].numpy(), p[want.astype(np.int64)]), i
    bad = inputs[0].copy()
    bad[7, 1] = np.nan
    hb = torch.from_numpy(bad).pin_memory()
    build_round_robin_host(hb, hout[0], hperm[0])
    with pytest.raises(ValueError, match="finite"):
        host_join()
    build_round_robin_host(hin[1], hout[1], hperm[1])  # the flag was cleared
    host_join()


def test_pipelined_host_builds_widest():
    """lbkd_build_widest_host: pipelined host-buffer widest builds, each exact
    (permutation and split dims) against the oracle."""
    from paper_2211_00120_b200.builder import host_join
    from paper_2211_00120_b200.widest import build_widest_host

    n, k = 200003, 3
    inputs = [datagen.make(kind, n, k, seed=s) for s, kind in enumerate(("clustered", "uniform", "ties"))]
    hin = [torch.from_numpy(p).pin_memory() for p in inputs]
    hout = [torch.empty((n, k), dtype=torch.float32).pin_memory() for _ in inputs]
    hperm = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in inputs]
    hdims = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in inputs]
    for i in range(len(inputs)):
        build_widest_host(hin[i], hout[i], hperm[i], hdims[i])
    host_join()
    for i, p in enumerate(inputs):
        wp, wd = oracle.build_widest(p)
        assert np.array_equal(hperm[i].numpy().view(np.uint32), wp), i
        assert np.array_equal(hdims[i].numpy(), wd), i
        assert np.array_equal(hout[i].numpy(), p[wp.astype(np.int64)]), i


@pytest.mark.parametrize("n", [5000, 70001, 1 << 20])
def test_selection_subtree_kernel_for_round_robin(n):
    """The in-CTA selection kernel (default for widest) is bit-exact for
    round-robin too, including tie-heavy input and small trees."""
    from paper_2211_00120_b200 import _native

    _native.set_subtree_kernel("selection")
    try:
        for kind, k in (("uniform", 3), ("ties", 2), ("clustered", 4), ("signed_zero", 3)):
            pts = datagen.make(kind, n, k, seed=n + 3 * k)
            _, perm = gpu_rr(pts)
            assert np.array_equal(perm, oracle.build_rr(pts)), (kind, n, k)
    finally:
        _native.set_subtree_kernel("default")


def test_fused_histogram_flush_path():
    """The partition's fused next-level histogram keeps two 16-bit bins per
    warp-private word and flushes them at least every 255 subtiles; at test
    sizes a warp never reaches 255, so LBKD_HFLUSH_EVERY=1 forces the flush
    path on every subtile -- the builds must stay bit-exact."""
    import subprocess
    import sys

    code = r'''
import numpy as np, torch
import paper_2211_00120_b200 as kd
from paper_2211_00120_b200 import datagen
from oracle import oracle
for kind in ("uniform", "ties", "clustered"):
    pts = datagen.make(kind, 1_500_003, 3, seed=11)
    d = torch.from_numpy(pts).cuda()
    _, perm = kd.build_round_robin_cuda(d)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), oracle.build_rr(pts)), ("rr", kind)
    _, perm, dims = kd.build_widest_cuda(d)
    wp, wd = oracle.build_widest(pts)
    assert np.array_equal(perm.cpu().numpy().view(np.uint32), wp), ("widest", kind)
    assert np.array_equal(dims.cpu().numpy(), wd), ("widest dims", kind)
print("OK")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LBKD_HFLUSH_EVERY="1", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
