"""pytest plugin: run the REFERENCE's own test files against the drop-in.

This is the import swap of INTEGRATION.md applied to an unmodified reference
install (baseline/_ref, git-ignored): every build / query entry point of the
reference package ``lbkd`` is rebound to this repo's CUDA implementation
before the reference's tests are collected, so the tests exercise the B200
path while their oracles (verify.reference_build, verify.check_valid,
brute-force scans, treemath) stay the reference's own:

    lbkd.build_round_robin / builder.build_round_robin / verify.build_round_robin
                                 -> paper_2211_00120_b200.build_round_robin
    lbkd.build_widest / widest.build_widest -> paper_2211_00120_b200.build_widest
    lbkd.knn / queries.knn, lbkd.radius_query / queries.radius_query
                                 -> paper_2211_00120_b200.knn / radius_query

Used by tests/test_gpu_dropin.py:  pytest -p tests.dropin_swap <ref tests>
"""

import os

import lbkd
import lbkd.builder
import lbkd.queries
import lbkd.verify
import lbkd.widest

import paper_2211_00120_b200 as ours

SWAPPED = []


def _swap(module, name, new):
    setattr(module, name, new)
    SWAPPED.append(f"{module.__name__}.{name}")


def pytest_configure(config):
    _swap(lbkd, "build_round_robin", ours.build_round_robin)
    _swap(lbkd.builder, "build_round_robin", ours.build_round_robin)
    _swap(lbkd.verify, "build_round_robin", ours.build_round_robin)
    _swap(lbkd, "build_widest", ours.build_widest)
    _swap(lbkd.widest, "build_widest", ours.build_widest)
    _swap(lbkd, "knn", ours.knn)
    _swap(lbkd.queries, "knn", ours.knn)
    _swap(lbkd, "radius_query", ours.radius_query)
    _swap(lbkd.queries, "radius_query", ours.radius_query)
    # create the CUDA context and load the library once, outside any test
    ours.build_round_robin([[1.0, 2.0], [3.0, 4.0], [0.5, 0.25]])
    report = os.environ.get("LBKD_DROPIN_REPORT")
    if report:
        with open(report, "w") as f:
            f.write("\n".join(SWAPPED) + "\n")


def pytest_report_header(config):
    return "drop-in swap: " + ", ".join(SWAPPED)
