"""Probe the host numpy arithmetic the reference's bits depend on.

The reference computes squared distances with np.einsum('ij,ij->i')
(kmeans.py:159, :484, :497).  In 3D numpy's SIMD kernels do not sum the three
products left to right; the order depends on the host build.
The kernels take the order as a parameter; this module finds it once per
process by comparing einsum against the three candidate orders.
"""

from __future__ import annotations

import functools

import numpy as np

ORDERS3 = {0: "(x+y)+z", 1: "(x+z)+y", 2: "(y+z)+x"}


@functools.lru_cache(maxsize=None)
def einsum_order3() -> int:
    rng = np.random.default_rng(12345)
    diff = rng.random((20000, 3)) - 0.5
    diff *= rng.uniform(0.1, 10.0, (20000, 1))
    got = np.einsum("ij,ij->i", diff, diff)
    sq = diff * diff
    cands = {
        0: (sq[:, 0] + sq[:, 1]) + sq[:, 2],
        1: (sq[:, 0] + sq[:, 2]) + sq[:, 1],
        2: (sq[:, 1] + sq[:, 2]) + sq[:, 0],
    }
    hits = [o for o, v in cands.items() if np.array_equal(v, got)]
    if len(hits) != 1:
        raise RuntimeError(
            "host numpy einsum('ij,ij->i') matches none of the supported 3D summation "
            "orders; device distances would not be bit-identical to the reference"
        )
    # the 2D case has a single order (commutativity); check it anyway
    d2 = diff[:, :2]
    if not np.array_equal(np.einsum("ij,ij->i", d2, d2), sq[:, 0] + sq[:, 1]):
        raise RuntimeError("host numpy einsum 2D order is not dx^2 + dy^2")
    return hits[0]
