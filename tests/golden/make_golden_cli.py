"""Golden files for the CLI / CSV formats, produced by the reference's CLI.

Runs ONLY in the authoring container (reference at /root/reference):

    NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_golden_cli.py

Writes tests/golden/cli/: points.csv (float32-representable coordinates +
payload), the reference's ``lbkd build`` outputs tree_rr.csv / tree_widest.csv,
its ``lbkd query`` stdout for a few queries (queries.json), and the error
messages of malformed point / tree files (errors.json).
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nc")

from lbkd import cli  # noqa: E402  (the reference)

MALFORMED = {
    "points_short_row.csv": ("points", "1,2\n3\n"),
    "points_bad_coord.csv": ("points", "1,2\n\nx,4\n"),
    "points_bad_payload.csv": ("points_payload", "1,2,7\n3,4,z\n"),
    "tree_no_coord.csv": ("tree", "x,y\n1,2\n"),
    "tree_bad_column.csv": ("tree", "coord_0,coord_1,weight\n1,2,3\n"),
    "tree_short_row.csv": ("tree", "coord_0,coord_1\n1,2\n3\n"),
    "tree_bad_dim.csv": ("tree", "coord_0,coord_1,split_dim\n1,2,0\n3,4,2\n"),
    "tree_nonfinite.csv": ("tree", "coord_0,coord_1\n1,2\ninf,4\n"),
}


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        rc = cli.main(argv)
    return rc, buf.getvalue()


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(4242)
    n, k = 300, 3
    pts = np.floor(rng.random((n, k)) * 64 * 16) / 16  # multiples of 1/16: float32-exact, many ties
    pts[rng.integers(0, n, 20)] = pts[rng.integers(0, n, 20)]
    payload = rng.integers(-1000, 1000, n)
    with open(os.path.join(OUT, "points.csv"), "w") as fh:
        for row, p in zip(pts, payload):
            fh.write(",".join(repr(float(v)) for v in row) + f",{int(p)}\n")
    res = {}
    for mode, name in (("round-robin", "tree_rr.csv"), ("widest", "tree_widest.csv")):
        rc, out = run(["build", "--input", os.path.join(OUT, "points.csv"), "--dims", "3", "--mode", mode,
                       "--output", os.path.join(OUT, name), "--payload"])
        assert rc == 0, out
        res[f"build {mode}"] = out.replace(OUT + "/", "")
        for q in ("10,20,30", "0,0,0", "32.5,12.0625,40"):
            for flag, val in (("--knn", "5"), ("--knn", "40"), ("--radius", "9.5"), ("--radius", "0")):
                rc, out = run(["query", "--tree", os.path.join(OUT, name), "--point", q, flag, val])
                assert rc == 0
                res[f"{name} {q} {flag} {val}"] = out
    with open(os.path.join(OUT, "queries.json"), "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)
    errs = {}
    for fname, (kind, text) in MALFORMED.items():
        path = os.path.join("/tmp", fname)
        with open(path, "w") as fh:
            fh.write(text)
        try:
            if kind == "tree":
                cli.read_tree(path)
            else:
                cli.read_points(path, 2, kind == "points_payload")
            errs[fname] = None
        except ValueError as e:
            errs[fname] = str(e).replace("/tmp/", "")
    with open(os.path.join(OUT, "errors.json"), "w") as fh:
        json.dump({"files": {f: t for f, (_, t) in MALFORMED.items()},
                   "kinds": {f: kd for f, (kd, _) in MALFORMED.items()}, "errors": errs}, fh, indent=1)
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
