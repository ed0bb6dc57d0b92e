"""Helpers to load the committed golden fixtures (made by tests/golden/make_golden.py)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def index():
    with open(os.path.join(GOLDEN, "index.json")) as f:
        return json.load(f)


def load(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def sha(arr, dtype):
    return np.frombuffer(hashlib.sha256(np.asarray(arr).astype(dtype).tobytes()).digest(), np.uint8)


def host_matches_golden_numerics():
    """True when this host's numpy pow/exp/einsum bits equal those the fixtures were made with."""
    import cases

    return cases.numerics_fingerprint() == index()["env"]
