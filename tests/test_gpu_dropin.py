"""The reference's own test files, unchanged, against the drop-in.

baseline/_ref holds the unmodified reference package and a copy of its
pkg/tests (git-ignored; installed with the pip command in DESIGN.md §5).
tests/dropin_swap.py rebinds the reference's build and query entry points to
this repo's CUDA path (the INTEGRATION.md import swap); the reference's
oracles stay its own.  test_verify.py / test_cli.py are not run: they
monkeypatch the reference's internal phases (sort_phase, the CLI's selftest
fixtures), which the swapped build does not use by design.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
FILES = ["test_builder.py", "test_widest.py", "test_acceptance.py", "test_queries.py", "test_treemath.py"]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")), reason="baseline/_ref/tests not installed")
def test_reference_test_suite_passes_against_dropin(tmp_path):
    report = str(tmp_path / "swapped.txt")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]), NUMBA_CACHE_DIR="/tmp/lbkd_dropin_numba",
               LBKD_DROPIN_REPORT=report)
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "tests.dropin_swap", "-p", "no:cacheprovider",
           "--rootdir", os.path.join(REF, "tests"), "-o", "addopts="] + [os.path.join(REF, "tests", f) for f in FILES]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1800)
    out = r.stdout + r.stderr
    with open(os.path.join(ROOT, "gpurun_out", "dropin_reference_tests.txt") if os.path.isdir(
            os.path.join(ROOT, "gpurun_out")) else os.devnull, "w") as f:
        f.write(out)
    swapped = open(report).read().split() if os.path.exists(report) else []
    assert "lbkd.builder.build_round_robin" in swapped and "lbkd.widest.build_widest" in swapped, out[-3000:]
    assert r.returncode == 0, out[-6000:]
    assert " passed" in out and " failed" not in out, out[-3000:]
