"""Generate golden fixtures from the LIVE reference (run in the dev container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs are not stored: every case is regenerated from its seeded recipe
(`tests/golden/cases.py`), which only uses numpy's PCG64 streams
(platform independent).  Outputs are written to `tests/golden/*.npz` plus
`tests/golden/index.json`.  The reference itself never travels to the GPU
box; these files do.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from geopart.geometry import BoundingBox, hilbert_keys  # noqa: E402
from geopart.kmeans import KMeansSettings, balanced_kmeans_points  # noqa: E402


def key_cases():
    out = {}
    for name, (pts, lo, hi, depth) in cases.key_inputs().items():
        out[name] = hilbert_keys(pts, BoundingBox(lo, hi), depth)
    return out


def partition_case(spec):
    pts, w = cases.partition_inputs(spec)
    settings = KMeansSettings(**spec["settings"])
    part, stats = balanced_kmeans_points(pts, w, settings, p=spec.get("p", 1), return_stats=True)
    st = stats.final_state
    recs = [vars(r) for r in stats.iterations]
    arrays = dict(
        assignment=part.assignment.astype(np.int32),
        centers=st.centers,
        influence=st.influence,
        block_weights=st.block_weights,
        empty_blocks=part.empty_blocks,
    )
    meta = dict(
        balance_failed=bool(part.balance_failed),
        converged=bool(stats.converged),
        audited_point_iterations=int(stats.audited_point_iterations),
        bound_violations=int(stats.bound_violations),
        skip_check_failures=int(stats.skip_check_failures),
        records=recs,
    )
    return arrays, meta


def sfc_case(spec):
    """Keys, SFC order and initial centers straight from the reference modules."""
    from geopart.kmeans import initial_center_positions
    from geopart.ranksim import RankWorld, global_sort_redistribute

    pts, w = cases.partition_inputs(spec)
    n, d = pts.shape
    depth = {2: 31, 3: 20}[d]
    world = RankWorld.from_points(pts, w, 1)
    box = BoundingBox(pts.min(axis=0), pts.max(axis=0))
    keys = hilbert_keys(pts, box, depth)
    world = global_sort_redistribute(world, [keys])
    order = world.shards[0].gids
    centers = world.shards[0].points[initial_center_positions(n, spec["settings"]["k"])]
    stride = max(1, n // 4096)
    return dict(
        keys_sha256=np.frombuffer(hashlib.sha256(keys.astype("<u8").tobytes()).digest(), np.uint8),
        order_sha256=np.frombuffer(
            hashlib.sha256(order.astype("<i4").tobytes()).digest(), np.uint8),
        keys_sample=keys[::stride],
        order_sample=order[::stride].astype(np.int32),
        stride=np.array([stride]),
        init_centers=centers,
    )


def main():
    index = {"env": cases.numerics_fingerprint(), "keys": [], "partitions": {}, "sfc": {}}
    kc = key_cases()
    np.savez_compressed(os.path.join(HERE, "keys.npz"), **kc)
    index["keys"] = sorted(kc)
    for spec in cases.PARTITION_CASES:
        arrays, meta = partition_case(spec)
        np.savez_compressed(os.path.join(HERE, f"part_{spec['name']}.npz"), **arrays)
        index["partitions"][spec["name"]] = meta
        print("partition", spec["name"], "iters", len(meta["records"]), flush=True)
    for spec in cases.SFC_CASES:
        arrays = sfc_case(spec)
        np.savez_compressed(os.path.join(HERE, f"sfc_{spec['name']}.npz"), **arrays)
        index["sfc"][spec["name"]] = True
        print("sfc", spec["name"], flush=True)
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
