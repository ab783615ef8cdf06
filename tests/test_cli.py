"""CLI and CSV formats against the reference CLI's own outputs
(tests/golden/cli/, made by tests/golden/make_golden_cli.py)."""

import contextlib
import io
import json
import os

import numpy as np
import pytest

from paper_2211_00120_b200 import KdTree, cli
from tests.golden_util import GOLDEN

CLI = os.path.join(GOLDEN, "cli")


def text(path):
    with open(path) as fh:
        return fh.read()


@pytest.mark.parametrize("name", ["tree_rr.csv", "tree_widest.csv"])
def test_tree_csv_round_trip(name, tmp_path):
    tree = cli.read_tree(os.path.join(CLI, name))
    assert tree.n == 300 and tree.k == 3 and (tree.split_dims is not None) == ("widest" in name)
    out = tmp_path / name
    cli.write_tree(str(out), tree, with_payload=True)
    assert text(out) == text(os.path.join(CLI, name))


def test_empty_tree_is_a_zero_byte_file(tmp_path):
    p = tmp_path / "empty.csv"
    cli.write_tree(str(p), KdTree(np.empty((0, 2)), np.empty(0, np.int64)))
    assert text(p) == ""
    assert cli.read_tree(str(p)).n == 0


def test_malformed_files_raise_the_reference_messages(tmp_path):
    spec = json.load(open(os.path.join(CLI, "errors.json")))
    for fname, body in spec["files"].items():
        path = tmp_path / fname
        path.write_text(body)
        kind = spec["kinds"][fname]
        with pytest.raises(ValueError) as e:
            if kind == "tree":
                cli.read_tree(str(path))
            else:
                cli.read_points(str(path), 2, kind == "points_payload")
        assert str(e.value).replace(str(tmp_path) + "/", "") == spec["errors"][fname]


def test_read_points_matches_file():
    coords, payload = cli.read_points(os.path.join(CLI, "points.csv"), 3, True)
    assert coords.shape == (300, 3) and payload.shape == (300,)
    assert np.array_equal(coords.astype(np.float32).astype(np.float64), coords)


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


@pytest.mark.gpu
def test_build_and_query_match_reference_cli(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    want = json.load(open(os.path.join(CLI, "queries.json")))
    for mode, name in (("round-robin", "tree_rr.csv"), ("widest", "tree_widest.csv")):
        out = tmp_path / name
        rc, msg = run(["build", "--input", os.path.join(CLI, "points.csv"), "--dims", "3", "--mode", mode,
                       "--output", str(out), "--payload"])
        assert rc == 0 and msg.replace(str(tmp_path) + "/", "") == want[f"build {mode}"]
        assert text(out) == text(os.path.join(CLI, name))
        for key, expect in want.items():
            if not key.startswith(name + " "):
                continue
            _, q, flag, val = key.split(" ")
            rc, got = run(["query", "--tree", str(out), "--point", q, flag, val])
            assert rc == 0 and got == expect, key


@pytest.mark.gpu
def test_bench_record(capsys):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    assert cli.main(["bench", "--n", "100000", "--dims", "3", "--reps", "2"]) == 0
    rec = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert {"n", "k", "mode", "seed", "reps", "millis", "device_millis", "mpts_per_s", "dtype"} <= set(rec)
    assert rec["n"] == 100000 and rec["device_millis"] > 0
