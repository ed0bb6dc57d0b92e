"""The hand-written device radix sort (csrc/radix.cu) through the C ABI gp_sort_pairs:
bit-exact against numpy's stable sort (= np.lexsort((gids, keys)), ranksim.py:158)
on every path -- the top-bits hybrid with its bucket-rank pass, the overflow
fallback (large buckets of equal high bits), small n, partial last tiles and
digits, and vals_in = NULL (value = input position)."""

import numpy as np
import pytest
import torch

from paper_1805_01208_b200 import _native as N


def _sort(keys: np.ndarray, vals: np.ndarray | None, bits: int):
    dev = torch.device("cuda")
    n = keys.shape[0]
    k = torch.from_numpy(keys.view(np.int64)).to(dev)
    v = torch.from_numpy(vals.view(np.int32)).to(dev) if vals is not None else None
    ko = torch.empty_like(k)
    vo = torch.empty(n, dtype=torch.int32, device=dev)
    k0 = k.clone()
    wsb = N.size_query("gp_sort_workspace_bytes", n)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    N.call("gp_sort_pairs", k.data_ptr(), v.data_ptr() if v is not None else None,
           ko.data_ptr(), vo.data_ptr(), n, bits, ws.data_ptr(), wsb,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(k, k0), "input keys modified"
    return ko.cpu().numpy().view(np.uint64), vo.cpu().numpy().view(np.uint32)


def _check(keys, bits, vals=None):
    n = keys.shape[0]
    ko, vo = _sort(keys, vals, bits)
    masked = keys & np.uint64((1 << bits) - 1) if bits < 64 else keys
    order = np.argsort(masked, kind="stable")
    exp_v = (vals if vals is not None else np.arange(n, dtype=np.uint32))[order]
    assert np.array_equal(vo, exp_v.astype(np.uint32))
    assert np.array_equal(ko, keys[order])


def _keys(kind: str, n: int, bits: int, rng) -> np.ndarray:
    if kind == "uniform":
        k = rng.integers(0, 1 << bits, n, dtype=np.uint64) if bits < 64 else \
            rng.integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2)
    elif kind == "clustered":  # a few hot high-bit regions with spread low bits
        hot = rng.integers(0, 1 << bits, 8, dtype=np.uint64)
        off = rng.integers(0, 1 << max(bits - 30, 1), n, dtype=np.uint64)
        k = (hot[rng.integers(0, 8, n)] & ~np.uint64((1 << max(bits - 30, 1)) - 1)) | off
    elif kind == "dups":  # few distinct keys: bucket overflow -> full-width fallback
        k = rng.integers(0, 1 << bits, 5, dtype=np.uint64)[rng.integers(0, 5, n)]
    elif kind == "equal":
        k = np.full(n, rng.integers(0, 1 << bits), dtype=np.uint64)
    elif kind == "sorted":
        k = np.sort(rng.integers(0, 1 << bits, n, dtype=np.uint64))
    else:
        raise ValueError(kind)
    return k.astype(np.uint64)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 100, 4095, 4096, 4097, 70001, (1 << 20) + 7])
@pytest.mark.parametrize("kind", ["uniform", "clustered", "dups", "sorted"])
def test_sort_pairs_matches_stable_sort(n, kind):
    rng = np.random.default_rng(n * 7 + len(kind))
    for bits in (62, 60):
        _check(_keys(kind, n, bits, rng), bits)


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [1, 5, 8, 9, 17, 31, 33, 64])
def test_sort_pairs_bit_widths(bits):
    rng = np.random.default_rng(bits)
    n = 300_000
    keys = rng.integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2) + \
        rng.integers(0, 2, n, dtype=np.uint64)
    _check(keys, bits)  # bits above key_bits are carried, not sorted on


@pytest.mark.gpu
def test_sort_pairs_explicit_vals_and_equal_keys():
    rng = np.random.default_rng(5)
    n = 200_003
    keys = _keys("equal", n, 62, rng)
    vals = rng.permutation(n).astype(np.uint32)
    _check(keys, 62, vals)
    keys = _keys("clustered", n, 62, rng)
    _check(keys, 62, vals)


@pytest.mark.gpu
def test_sort_pairs_large_hybrid():
    # 2^26 SFC-like keys: the hybrid path (3 top passes + bucket rank) at scale
    rng = np.random.default_rng(11)
    n = 1 << 26
    keys = rng.integers(0, 1 << 62, n, dtype=np.uint64)
    ko, vo = _sort(keys, None, 62)
    assert np.all(ko[1:] >= ko[:-1])
    sel = rng.integers(0, n, 1 << 16)
    assert np.array_equal(keys[vo[sel]], ko[sel])
    eq = ko[1:] == ko[:-1]
    assert np.all(vo[1:][eq] > vo[:-1][eq])
    assert np.array_equal(np.sort(vo), np.arange(n, dtype=np.uint32))
