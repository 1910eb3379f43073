"""(f1) The decay-window memory-allocation search is pinned to the reference.

``tests/golden/window/cases.json.gz`` holds the UNMODIFIED reference's
``decay_window_search`` (profiler.py:281-354) results -- made by
``tests/golden/make_window_golden.py`` -- for 525 synthetic throughput curves and for
every measured B200 curve under ``profiles/`` (``search_memory_allocation_measured``
on the GPU, replayed from its recorded samples).  This package's search must return
the identical document (lower / upper / chosen / samples / stop_error / warning).
"""

import gzip
import json
import os

import pytest

from paper_2503_02354_b200 import profiler

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(gzip.open(os.path.join(HERE, "golden", "window", "cases.json.gz"), "rt"))["cases"]


def _ours(case):
    if "curve" in case:
        sample = lambda c: case["curve"][c - 1]  # noqa: E731
    else:
        table = {int(n): float(t) for n, t in case["samples"]}
        sample = lambda c: table[c]  # noqa: E731
    return profiler.decay_window_search(sample, max_count=case["max_count"], initial_window=case["initial_window"],
                                        error_margin=case["error_margin"], fit_points=case["fit_points"],
                                        seed=case["seed"], choose=case["choose"]).to_doc()


def test_synthetic_curves_match_reference():
    synthetic = [c for c in CASES if "curve" in c]
    assert len(synthetic) >= 500
    bad = [c["name"] for c in synthetic if _ours(c) != c["expected"]]
    assert not bad, bad[:10]


@pytest.mark.parametrize("case", [c for c in CASES if "samples" in c], ids=lambda c: c["name"])
def test_measured_b200_search_matches_reference(case):
    """The reference, replaying the B200 samples, picks the same window and count as the
    measured search did on the GPU, and as this package's search does on the same samples."""
    assert case["expected"] == case["recorded"]
    assert _ours(case) == case["expected"]
