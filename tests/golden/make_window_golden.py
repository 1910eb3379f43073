"""Golden decay-window searches made by the UNMODIFIED reference (build container only).

    python tests/golden/make_window_golden.py

The reference's ``coesim.profiler.decay_window_search`` (profiler.py:281-354) is fed
throughput curves through its ``sample_throughput`` callback:

* synthetic curves over every expert count (rising, saturating, collapsing, flat,
  noisy, non-positive), across window / margin / fit-point / choose settings;
* every MEASURED B200 curve committed under ``profiles/*window_search*.json``
  (``profiler.search_memory_allocation_measured`` on the GPU): the reference replays
  the recorded samples (a count the B200 search never probed raises, so the window
  schedule itself is pinned too).

Output: ``tests/golden/window/cases.json.gz`` -- inputs and the reference's
``WindowSearchResult.to_doc()`` per case.  ``tests/test_window_search_golden.py``
checks ``paper_2503_02354_b200.profiler.decay_window_search`` against it on CPU.
"""

from __future__ import annotations

import glob
import gzip
import json
import math
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from coesim.profiler import decay_window_search  # noqa: E402


def synthetic_cases():
    rng = random.Random(2503)
    shapes = {
        "rising": lambda c, m: 100.0 + 5.0 * c,
        "saturating": lambda c, m: 1000.0 * (1.0 - math.exp(-c / (0.3 * m))),
        "knee": lambda c, m: 10.0 * c if c < 0.6 * m else 6.0 * m - 20.0 * (c - 0.6 * m),
        "collapse": lambda c, m: 500.0 + c if c < 0.5 * m else 50.0,
        "flat": lambda c, m: 321.0,
        "falling": lambda c, m: 1000.0 - 3.0 * c,
        "to_zero": lambda c, m: max(0.0, 400.0 - 9.0 * c),
    }
    cases = []
    for name, f in shapes.items():
        for max_count in (1, 7, 59, 148, 300):
            for initial_window in (1, 15, 40, 100, 120):
                for error_margin, fit_points, choose in ((0.05, 4, "random"), (0.02, 3, "midpoint"),
                                                         (0.2, 2, "random")):
                    noise = [rng.uniform(-0.03, 0.03) for _ in range(max_count)]
                    curve = [f(c, max_count) * (1.0 + (noise[c - 1] if name != "flat" else 0.0))
                             for c in range(1, max_count + 1)]
                    cases.append({"name": f"{name}-m{max_count}-w{initial_window}-e{error_margin}-f{fit_points}"
                                          f"-{choose}", "curve": curve, "max_count": max_count,
                                  "initial_window": initial_window, "error_margin": error_margin,
                                  "fit_points": fit_points, "choose": choose, "seed": rng.randrange(1 << 30)})
    return cases


def measured_cases():
    cases = []
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*window_search*.json"))):
        doc = json.load(open(path))
        m = doc.get("measured")
        if not m:
            continue
        params = doc.get("search", {})
        cases.append({"name": "measured:" + os.path.basename(path), "samples": m["throughput_samples"],
                      "max_count": params.get("max_count", max(n for n, _ in m["throughput_samples"])),
                      "initial_window": params.get("initial_window", 15),
                      "error_margin": params.get("error_margin", 0.05), "fit_points": params.get("fit_points", 3),
                      "choose": params.get("choose", "random"), "seed": params.get("seed", doc.get("seed", 0)),
                      "recorded": m})
    return cases


def run(case):
    if "curve" in case:
        sample = lambda c: case["curve"][c - 1]  # noqa: E731
    else:
        table = {int(n): float(t) for n, t in case["samples"]}
        sample = lambda c: table[c]  # noqa: E731
    res = decay_window_search(sample, max_count=case["max_count"], initial_window=case["initial_window"],
                              error_margin=case["error_margin"], fit_points=case["fit_points"], seed=case["seed"],
                              choose=case["choose"])
    return res.to_doc()


def main():
    cases = synthetic_cases() + measured_cases()
    for case in cases:
        case["expected"] = run(case)
    out = os.path.join(HERE, "window", "cases.json.gz")
    with gzip.open(out, "wt") as fh:
        json.dump({"generator": "reference coesim.profiler.decay_window_search", "cases": cases}, fh)
    print(len(cases), "cases ->", out)


if __name__ == "__main__":
    main()
