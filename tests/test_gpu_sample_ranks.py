"""gp_sample_ranks reproduces numpy.random.default_rng(seed).permutation(n) bit for bit
(kmeans.py:564-567).  Edge sizes: 1, 2, powers of two and their neighbours, large n."""
import numpy as np
import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2, 3, 5, 31, 32, 33, 100, 1000, 4095, 4096, 4097, 65537, 200_000,
                               (1 << 17) * 3 // 2 + 1,
                               1_000_003, (1 << 22) + 5])
@pytest.mark.parametrize("seed", [0, 7])
def test_device_permutation_matches_numpy(n, seed):
    if not has_cuda():
        pytest.fail("CUDA device required")
    import torch

    from paper_1805_01208_b200.kmeans import sample_ranks_device

    dev = torch.device("cuda")
    rank = sample_ranks_device(n, seed, dev, torch.cuda.current_stream().cuda_stream)
    perm = np.random.default_rng(seed).permutation(n)
    want = np.empty(n, dtype=np.int64)
    want[perm] = np.arange(n)
    assert np.array_equal(rank.cpu().numpy(), want)


def test_device_permutation_large():
    import torch

    from paper_1805_01208_b200.kmeans import sample_ranks_device

    n = (1 << 26) + 12345
    rank = sample_ranks_device(n, 3, torch.device("cuda"), torch.cuda.current_stream().cuda_stream)
    perm = np.random.default_rng(3).permutation(n)
    got = rank.cpu().numpy()
    assert np.array_equal(got[perm], np.arange(n, dtype=got.dtype))
