"""Parity on the BASELINE configurations at their stated sizes.

* C2, C3, C4: the complete partition against fixtures made by the LIVE reference
  (`tests/golden/make_golden_configs.py`, `geopart.kmeans.balanced_kmeans_points`
  on the SURVEY §8d recipes): labels (sha256 + a strided sample), the final
  k-sized state, the flags and every per-iteration record, bit for bit.  Bit-exact
  is stricter than north_star's "identical outside 1e-9 near-ties, centers within
  1e-9 relative".
* C5 (2^30 points, k = 16384; the reference cannot run it), per SURVEY §8c:
  Hilbert keys of a 2^24-point random subsample against the oracle under the
  global box; the full SFC sort checked through size-independent properties
  (sorted keys, gids a permutation, payload travelled with its gid); the final
  partition's balance (imbalance <= epsilon, recomputed from the labels) and an
  exact-argmin audit of random subsamples of the final state (2^16 points against
  the oracle, 2^20 points against an independent fp64 torch checker that the
  oracle pins); and the warm-up permutation at n = 2^30 against numpy.
"""
import json
import os

import numpy as np
import pytest

import cases  # noqa: F401  (tests/golden on sys.path)
import golden_io
from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if has_cuda():
    import torch

    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points
    from paper_1805_01208_b200.kmeans import DevicePartitioner, sample_ranks_device
    from paper_1805_01208_b200.workloads import CONFIGS, GENERATORS, c5_device

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("CUDA device required for -m gpu tests")


def _oracle():
    from oracle import geographer_oracle as O

    return O


def _meta(name):
    with open(os.path.join(GOLDEN, f"cfg_{name}.json")) as f:
        return json.load(f)


def _compare_records(got, want):
    assert len(got) == len(want)
    for g, w in zip(got, want):
        g = vars(g)
        for key in ("phase", "active_points", "balance_rounds", "imbalance", "total_decisions",
                    "max_move"):
            assert g[key] == w[key], (key, g[key], w[key])
        assert g["objective"] == pytest.approx(w["objective"], rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_config_full_size_vs_reference_golden(name):
    """BASELINE configs[1..3] end to end at full size against the live reference."""
    if not os.path.exists(os.path.join(GOLDEN, f"cfg_{name}.json")):
        pytest.fail(f"fixture cfg_{name} missing: run tests/golden/make_golden_configs.py")
    meta = _meta(name)
    c = CONFIGS[name]
    pts, w = GENERATORS[name](seed=0)
    s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
    part, stats = balanced_kmeans_points(pts, w, s, return_stats=True)
    st = stats.final_state
    if meta["env"] != _oracle_free_fingerprint():
        # this host's numpy pow/exp/einsum bits differ from the fixture host's, so the
        # reference itself would give other bits here: compare with the oracle run here
        if name == "C4":
            pytest.skip("numerics fingerprint differs from the fixture host; the C4 oracle "
                        "run (~20 min) is not repeated here")
        O = _oracle()
        r = O.run(pts, w, O.Knobs(k=c["k"], epsilon=c["epsilon"], seed=0), scan_chunks=256)
        assert np.array_equal(part.assignment, r.assignment)
        assert np.array_equal(st.centers, r.centers)
        assert np.array_equal(st.influence, r.influence)
        _compare_records(stats.iterations, r.records)
        return
    gold = golden_io.load(f"cfg_{name}")
    a = part.assignment.astype(np.int32)
    stride = int(gold["stride"][0])
    sample_bad = int(np.count_nonzero(a[::stride] != gold["assignment_sample"]))
    assert sample_bad == 0, f"{sample_bad} sampled labels differ"
    assert np.array_equal(golden_io.sha(a, "<i4"), gold["assignment_sha256"])
    assert np.array_equal(st.centers, gold["centers"])
    assert np.array_equal(st.influence, gold["influence"])
    assert np.array_equal(st.block_weights, gold["block_weights"])
    assert np.array_equal(part.empty_blocks, gold["empty_blocks"])
    assert part.balance_failed == meta["balance_failed"]
    assert stats.converged == meta["converged"]
    _compare_records(stats.iterations, meta["records"])
    assert _oracle().imbalance(st.block_weights) <= c["epsilon"] or meta["balance_failed"]


def _oracle_free_fingerprint():
    return cases.numerics_fingerprint()


# ------------------------------------------------------------------------ C5
def _torch_argmin(P, centers, infl, chunk=4096):
    """Independent exact checker: the reference's per-pair fp64 arithmetic
    (diff, separately rounded squares summed x then y, correctly rounded sqrt and
    division; one eager op per kernel, so nothing is contracted into FMA) and
    argmin's first-minimum tie-break."""
    C = torch.from_numpy(centers).cuda()
    f = torch.from_numpy(infl).cuda()
    out = []
    for s in range(0, P.shape[0], chunk):
        p = P[s:s + chunk]
        dx = p[:, None, 0] - C[None, :, 0]
        dy = p[:, None, 1] - C[None, :, 1]
        q = dx * dx
        q = q + dy * dy
        out.append(torch.argmin(torch.sqrt(q) / f[None, :], dim=1))
    return torch.cat(out)


@pytest.fixture(scope="module")
def c5_run():
    c = CONFIGS["C5"]
    n, k = c["n"], c["k"]
    X = c5_device(n=n, seed=0)                    # (2, n) device SoA
    pts = X.t()
    eng = DevicePartitioner(KMeansSettings(k=k, epsilon=c["epsilon"], seed=0), keep_keys=True)
    eng.bootstrap(pts, None)
    # ---- SFC stage at full size (size-independent properties) + a key subsample
    ks = eng.keys_sorted
    sfc = {}
    sfc["sorted"] = bool((ks[1:] >= ks[:-1]).all().item())
    g = eng.gids.long()
    seen = torch.zeros(n, dtype=torch.uint8, device=g.device)
    seen[g] = 1
    sfc["perm"] = bool(seen.all().item()) and int(g.min().item()) == 0
    del seen
    sfc["payload"] = bool(torch.equal(eng.X[:, 0], X[0][g]) and torch.equal(eng.X[:, 1], X[1][g]))
    rng = np.random.default_rng(5)
    pos = np.sort(rng.choice(n, 1 << 24, replace=False))
    pos_d = torch.from_numpy(pos).cuda()
    sfc["sub_pts"] = eng.X[pos_d].cpu().numpy()
    sfc["sub_keys"] = ks[pos_d].cpu().numpy().view(np.uint64)
    sfc["box"] = (eng.box.lo.copy(), eng.box.hi.copy())
    eng.keys_sorted = None
    del ks, g, pos_d
    labels, stats = eng.run()
    return dict(X=X, labels=labels, stats=stats, sfc=sfc, k=k, eps=c["epsilon"], n=n)


def test_c5_sfc_stage(c5_run):
    sfc = c5_run["sfc"]
    assert sfc["sorted"] and sfc["perm"] and sfc["payload"]
    O = _oracle()
    lo, hi = sfc["box"]
    want = O.hilbert_keys(sfc["sub_pts"], lo, hi, 31)
    assert np.array_equal(sfc["sub_keys"], want)


def test_c5_balance(c5_run):
    st = c5_run["stats"]
    k, eps = c5_run["k"], c5_run["eps"]
    assert not st.balance_failed
    bw = torch.bincount(c5_run["labels"], minlength=k).cpu().numpy().astype(np.float64)
    assert np.array_equal(bw, st.final_state.block_weights)
    assert _oracle().imbalance(bw) <= eps


def test_c5_exact_argmin_subsamples(c5_run):
    st = c5_run["stats"].final_state
    X, labels, n = c5_run["X"], c5_run["labels"], c5_run["n"]
    rng = np.random.default_rng(11)
    ids = np.sort(rng.choice(n, 1 << 20, replace=False))
    ids_d = torch.from_numpy(ids).cuda()
    P = torch.stack([X[0][ids_d], X[1][ids_d]], dim=1)
    got = labels[ids_d]
    chk = _torch_argmin(P, st.centers, st.influence)
    # pin the torch checker to the oracle on the first 2^16 sample points
    O = _oracle()
    sub = P[:1 << 16].cpu().numpy()
    assert np.array_equal(chk[:1 << 16].cpu().numpy(),
                          O.brute_labels_blocked(sub, st.centers, st.influence))
    bad = int((chk != got).sum().item())
    assert bad == 0, f"{bad} of 2^20 sampled points are not at the exact argmin"


def test_sample_ranks_at_2e30_vs_numpy():
    """gp_sample_ranks at the C5 size (the bench's warm-up order) against numpy."""
    n = 1 << 30
    rank = sample_ranks_device(n, 0, torch.device("cuda"), torch.cuda.current_stream().cuda_stream)
    got = rank.cpu().numpy()
    del rank
    perm = np.random.default_rng(0).permutation(n)
    assert np.array_equal(got[perm], np.arange(n, dtype=got.dtype))
