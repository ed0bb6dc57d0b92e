"""The reference's own tests of the path and of the formats / metrics either side of it
(pkg/tests/test_kmeans.py, test_acceptance.py, test_estimators.py, test_cli.py,
test_fileio.py, test_metrics.py, test_graph.py) run against the B200 entry points through
the INTEGRATION.md shim (tools/ref_suite.py). Needs the git-ignored copies `baseline/_ref`
and `baseline/_ref_tests` that `__graft_entry__.build()` makes; skipped without them."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_reference_suite_through_shim(tmp_path):
    if not os.path.isfile(os.path.join(ROOT, "baseline", "_ref_tests", "conftest.py")) or \
            not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "geopart")):
        pytest.skip("baseline/_ref or baseline/_ref_tests missing (made by build())")
    out = tmp_path / "suite.json"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ref_suite.py"),
                        "--tests", os.path.join(ROOT, "baseline", "_ref_tests"),
                        "--out", str(out)], capture_output=True, text=True, timeout=1500)
    assert out.exists(), r.stdout[-3000:] + r.stderr[-3000:]
    s = json.loads(out.read_text())
    assert s["b200_calls"]["balanced_kmeans_points"] > 0
    for name in ("load_metis_graph", "read_partition", "write_partition", "evaluate",
                 "edge_cut", "comm_volumes", "block_diameter_lower_bounds",
                 "GeometricGraph.validate"):
        assert s["b200_calls"].get(name, 0) > 0, name
    assert s["outcomes"].get("failed", 0) == 0, s["failed"]
    assert r.returncode == 0, r.stdout[-3000:]
