"""The seeded input generator (datagen/): shape and statistics of the paper's workloads
(P:2003-2010 random walks, z-normalised P:326; P:2434-2436 noise queries)."""
import numpy as np
import pytest
import torch

import datagen


def test_walks_are_znormalised_random_walks():
    X = datagen.walks_cpu(0, 2000, 256)
    assert X.dtype == np.float32 and X.shape == (2000, 256)
    assert np.allclose(X.mean(1), 0, atol=1e-5)
    assert np.allclose(X.std(1), 1, atol=1e-4)
    # the walk's increments are i.i.d. N(0,1) up to the per-row z-normalisation scale
    raw = np.cumsum(datagen._normals(0, np.arange(2000), datagen.STREAM_WALK, 256), axis=1)
    inc = np.diff(raw, axis=1).ravel()
    assert abs(inc.mean()) < 0.01 and abs(inc.std() - 1) < 0.01
    # z-normalised raw walk reproduces the stored rows
    mu, sd = raw.mean(1, keepdims=True), raw.std(1, keepdims=True)
    assert np.allclose((raw - mu) / sd, X, atol=1e-5)


def test_counter_based_sharding():
    """Row r is the same whatever shard generates it (counter = row index)."""
    a = datagen.walks_cpu(0, 300, 64)
    b = datagen.walks_cpu(100, 50, 64)
    assert np.array_equal(a[100:150], b)
    assert not np.array_equal(datagen.walks_cpu(0, 5, 64, seed=1), a[:5])


def test_noisy_queries_shape():
    N = 1000
    Q = datagen.noisy_queries_cpu(30, 128, N, sigma=0.1)
    rows = datagen.noisy_rows(30, N)
    assert np.all((rows >= 0) & (rows < N))
    src = datagen.walks_cpu(0, N, 128)[rows]
    assert np.allclose(Q.mean(1), 0, atol=1e-5) and np.allclose(Q.std(1), 1, atol=1e-4)
    resid = (Q - src).std(1)
    assert np.all((resid > 0.05) & (resid < 0.2))  # ~ sigma after re-z-normalisation


@pytest.mark.gpu
def test_cuda_generator_matches_numpy_twin():
    X = torch.empty((512, 256), dtype=torch.float32, device="cuda:0")
    datagen.walks_cuda(X, 777)
    ref = datagen.walks_cpu(777, 512, 256)
    got = X.cpu().numpy()
    assert np.allclose(got, ref, rtol=0, atol=2e-6)
    assert np.mean(got == ref) > 0.99
    Q = torch.empty((16, 128), dtype=torch.float32, device="cuda:0")
    datagen.noisy_queries_cuda(Q, 100_000)
    assert np.allclose(Q.cpu().numpy(), datagen.noisy_queries_cpu(16, 128, 100_000), atol=2e-6)
