"""Run the reference's OWN hot-path test files against the B200 entry points.

This is the INTEGRATION.md shim exercised for real: the unmodified reference package
(`baseline/_ref`, installed by `__graft_entry__.build()`) is imported, and its
`geopart.kmeans.balanced_kmeans_points` / `balanced_kmeans` are replaced by this
package's, exactly as the one-line shim at the end of `geopart/kmeans.py` would do
(every module that bound the names at import time -- `geopart`, `geopart.estimators`,
`geopart.cli` -- sees the B200 functions). Then pytest runs the reference's own tests:

* `test_kmeans.py`      -- `pkg/tests/test_kmeans.py:99-183` (exact argmin, balance,
                           p-invariance, sample schedule) and the rest of the file;
* `test_acceptance.py`  -- ACCEPT-01..10 (`:108-231`: exact argmin, audit, convergence,
                           p-invariance), whose partitions now come from the GPU;
* `test_estimators.py`  -- `GeographerPartitioner.fit` through the shim;
* `test_cli.py`         -- `geopart partition --algo geographer` through the shim;
* `test_fileio.py`, `test_metrics.py`, `test_graph.py` -- the formats and metrics either
                           side of the path: the readers, the
                           partition writer, the metrics and `GeometricGraph.validate`
                           are replaced by the B200 ones (`integration.install_formats`).

The test files are read from `--tests` (default: `/root/reference/pkg/tests` where it
exists, else `baseline/_ref_tests`, the git-ignored copy `build()` makes so that it
travels to the GPU box with `baseline/_ref`). Nothing from the reference is committed.

The run FAILS if the B200 entry points were never called (the shim did not take).
Usage: python tools/ref_suite.py [--tests DIR] [--out FILE] [pytest args...]
"""

from __future__ import annotations

import argparse
import json
import os
import shutil
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = ("test_kmeans.py", "test_acceptance.py", "test_estimators.py", "test_cli.py",
         "test_fileio.py", "test_metrics.py", "test_graph.py")


def tests_dir(arg: str | None) -> str | None:
    for d in (arg, "/root/reference/pkg/tests", os.path.join(ROOT, "baseline", "_ref_tests")):
        if d and os.path.isfile(os.path.join(d, "conftest.py")):
            return d
    return None


class Shim:
    """Route the reference's entry points to the B200 ones (the package's own
    `integration.install`, i.e. the INTEGRATION.md shim) and count the calls."""

    def __init__(self):
        self.calls = {"balanced_kmeans_points": 0, "balanced_kmeans": 0}

    def install(self):
        import geopart  # noqa: F401  (the reference, from baseline/_ref)
        import geopart.cli  # noqa: F401
        import geopart.estimators  # noqa: F401

        from paper_1805_01208_b200 import integration

        integration.install(counter=self.calls)
        integration.install_formats(counter=self.calls)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--tests", default=None)
    ap.add_argument("--out", default=None, help="write a JSON summary here")
    ap.add_argument("--files", default=",".join(SUITE))
    args, rest = ap.parse_known_args(argv)

    src = tests_dir(args.tests)
    if src is None:
        print("reference tests not found (run __graft_entry__.build() where /root/reference exists)")
        return 2
    ref_pkg = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_pkg, "geopart")):
        print("reference package not installed in baseline/_ref")
        return 2
    sys.path.insert(0, ref_pkg)
    sys.path.insert(0, ROOT)

    import pytest

    shim = Shim()
    shim.install()

    # a scratch copy: the reference tree is read-only and pytest writes caches
    work = tempfile.mkdtemp(prefix="ref_suite_")
    tdir = os.path.join(work, "tests")
    shutil.copytree(src, tdir)
    files = [os.path.join(tdir, f) for f in args.files.split(",") if f]
    cwd = os.getcwd()
    os.chdir(tdir)

    class Collect:
        def __init__(self):
            self.outcomes = {}

        def pytest_runtest_logreport(self, report):
            if report.when == "call" or (report.when == "setup" and report.outcome != "passed"):
                self.outcomes[report.nodeid] = report.outcome

    col = Collect()
    t0 = time.perf_counter()
    try:
        rc = pytest.main(["-q", "-p", "no:cacheprovider", "--rootdir", tdir, *rest, *files],
                         plugins=[col])
    finally:
        os.chdir(cwd)
        shutil.rmtree(work, ignore_errors=True)
    wall = time.perf_counter() - t0
    counts = {}
    for o in col.outcomes.values():
        counts[o] = counts.get(o, 0) + 1
    summary = {
        "tests_from": src, "files": args.files.split(","), "pytest_rc": int(rc),
        "outcomes": counts, "b200_calls": shim.calls, "wall_s": round(wall, 1),
        "failed": sorted(k for k, v in col.outcomes.items() if v == "failed"),
    }
    print(json.dumps(summary, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(summary, f, indent=1)
    if sum(shim.calls.values()) == 0:
        print("the B200 entry points were never called: the shim did not take")
        return 1
    return int(rc)


if __name__ == "__main__":
    sys.exit(main())
