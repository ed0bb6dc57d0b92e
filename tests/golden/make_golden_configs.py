"""Golden results of the LIVE reference on the BASELINE configs at full size.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_configs.py C2 C3 C4

Runs `geopart.kmeans.balanced_kmeans_points` (`kmeans.py:502-512`) on the
seeded recipes of SURVEY §8d (`paper_1805_01208_b200/workloads.py`) and stores,
per config, `tests/golden/cfg_<C>.npz`:

* `assignment_sha256` of the int32 labels in original vertex order, plus every
  `stride`-th label (so a mismatch can be located and counted);
* the k-sized final state (centers, influence, block weights) in full;
* `tests/golden/cfg_<C>.json`: flags, the per-iteration records and the host
  numerics fingerprint (`cases.numerics_fingerprint`).

`p` only shards the simulated ranks; results are p-invariant
(`test_acceptance.py:213-231`), so the large configs use p=256, which is the
fastest setting of the reference there.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from geopart.kmeans import KMeansSettings, balanced_kmeans_points  # noqa: E402

sys.path.insert(0, os.path.join(HERE, "..", ".."))
from paper_1805_01208_b200.workloads import CONFIGS, GENERATORS  # noqa: E402

P = {"C1": 1, "C2": 1, "C3": 256, "C4": 256}
STRIDE = {"C1": 1, "C2": 16, "C3": 16, "C4": 64}


def run(name):
    cfg = CONFIGS[name]
    pts, w = GENERATORS[name](seed=0)
    settings = KMeansSettings(k=cfg["k"], epsilon=cfg["epsilon"], seed=0)
    t0 = time.perf_counter()
    part, stats = balanced_kmeans_points(pts, w, settings, p=P[name], return_stats=True)
    wall = time.perf_counter() - t0
    a = part.assignment.astype(np.int32)
    st = stats.final_state
    np.savez_compressed(
        os.path.join(HERE, f"cfg_{name}.npz"),
        assignment_sha256=np.frombuffer(hashlib.sha256(a.tobytes()).digest(), np.uint8),
        assignment_sample=a[::STRIDE[name]],
        stride=np.array([STRIDE[name]]),
        centers=st.centers, influence=st.influence, block_weights=st.block_weights,
        empty_blocks=part.empty_blocks)
    meta = dict(
        config=name, p=P[name], wall_s=wall, env=cases.numerics_fingerprint(),
        balance_failed=bool(part.balance_failed), converged=bool(stats.converged),
        records=[vars(r) for r in stats.iterations])
    with open(os.path.join(HERE, f"cfg_{name}.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(name, "wall", round(wall, 1), "s iters", len(meta["records"]), flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:]:
        run(name)
