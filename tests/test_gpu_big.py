"""BASELINE config 4 (1B clustered float3, round-robin) pinned bit-exact.

The expected permutation's sha256 in tests/golden/hashes.json comes from the
threaded recursive oracle (oracle/lbkd_recursive.cpp, restating
verify.reference_build, verify.py:121-168), which tests/golden/
make_golden_1b.py validated against every reference-generated hash first
(1M-100M, ties, +-0.0, clustered negatives, widest).

One GPU builds the whole tree; then the sharded decomposition of SURVEY.md
§8(e) for G = 2, 4, 8 -- top log2(G) levels (lbkd_build_rr_top), then every
subtree finished on its own (lbkd_build_rr_sub) -- must give the same bytes.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from tests.golden_util import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_00120_b200 as kd  # noqa: E402
from paper_2211_00120_b200 import datagen, multigpu  # noqa: E402
from paper_2211_00120_b200.verify import check_valid_cuda  # noqa: E402

KEY = "rr/clustered/n1000000000/k3/s0"


def _entry():
    h = json.load(open(os.path.join(GOLDEN, "hashes.json")))
    return h.get(KEY)


def _sha(t):
    return hashlib.sha256(np.ascontiguousarray(t).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def big():
    e = _entry()
    if e is None:
        pytest.skip("no 1B golden hash (run tests/golden/make_golden_1b.py)")
    free, _ = torch.cuda.mem_get_info()
    if free < 120e9:
        pytest.skip("needs ~120 GB of free device memory")
    pts = datagen.make(e["kind"], e["n"], e["k"], e["seed"])
    assert _sha(pts) == e["input_sha256"], "input generator drifted"
    d = torch.from_numpy(pts).cuda()
    del pts
    yield e, d
    del d
    torch.cuda.empty_cache()


def test_1b_single_gpu_matches_oracle_hash(big):
    e, d = big
    out, perm = kd.build_round_robin_cuda(d)
    p = perm.cpu().numpy().view(np.uint32)
    assert p[:64].tolist() == e["perm_head"]
    assert _sha(p) == e["perm_sha256"]
    assert torch.equal(out, d[perm.long()])
    assert check_valid_cuda(out) is None


@pytest.mark.parametrize("G", [2, 4, 8])
def test_1b_sharded_decomposition_bit_identical(big, G):
    e, d = big
    n, k = e["n"], e["k"]
    out, perm = kd.build_round_robin_cuda(d)
    ops = multigpu.CudaOps(0)
    top = multigpu.top_levels_for(G)
    sub = torch.empty((k + 1) * n, dtype=torch.int32, device="cuda")
    out2 = torch.full_like(out, float("nan"))
    perm2 = torch.full_like(perm, -1)
    ops.build_top(d, top, out2, perm2, sub, n)
    for sh in multigpu.shard_layout(n, top):
        ops.build_sub(sub[sh.offset:], n, n, k, top, sh.index, out2, perm2)
    torch.cuda.synchronize()
    assert torch.equal(perm2, perm)
    assert torch.equal(out2.view(torch.int32), out.view(torch.int32))
    del sub
    # recursive halving of the top levels (what build_round_robin_sharded runs)
    out2.fill_(float("nan"))
    perm2.fill_(-1)
    multigpu.serial_sharded_build(d, n, k, G, out=out2, perm=perm2)
    torch.cuda.synchronize()
    assert torch.equal(perm2, perm)
    assert torch.equal(out2.view(torch.int32), out.view(torch.int32))
    del out2, perm2
