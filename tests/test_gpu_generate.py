"""Device generator (csrc/generate.cu): the documented
Philox4x32-10 stream equals its numpy restatement (oracle.gen_*; Philox pinned
by the Random123 known-answer vectors in test_oracle.py) within float32
rounding, is prefix-stable, and keeps the reference generator's properties
(z-normalised, lag-1 autocorrelation > 0.8: test_generate.py:47-52)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2212_13297_b200 import generate

    return generate


@pytest.mark.parametrize("n", [256, 96, 33, 1, 1024])
def test_random_walks_match_restatement(G, oracle, n):
    D = G.random_walks_device(300, n, 5, start=17).cpu().numpy()
    R = oracle.gen_random_walks(17, 300, n, 5)
    assert np.abs(D - R).max() < 2e-5
    if n > 1:
        assert np.abs(D.mean(1)).max() < 1e-5 and np.abs(D.std(1) - 1).max() < 1e-5
    else:
        assert not D.any()  # a constant (one-point) series z-normalises to zeros


@pytest.mark.parametrize("n", [96, 256, 50])
def test_unit_gaussian_match_restatement(G, oracle, n):
    D = G.unit_gaussian_device(200, n, 2, start=65_530).cpu().numpy()
    R = oracle.gen_unit_gaussian(65_530, 200, n, 2)
    assert np.abs(D - R).max() < 1e-6
    assert np.abs(np.linalg.norm(D.astype(np.float64), axis=1) - 1).max() < 1e-6


def test_prefix_stable_and_seeded(G):
    A = G.random_walks_device(5000, 128, 3).cpu().numpy()
    B = G.random_walks_device(1000, 128, 3, start=2500).cpu().numpy()
    assert np.array_equal(A[2500:3500], B)
    C = G.random_walks_device(1000, 128, 4, start=2500).cpu().numpy()
    assert not np.array_equal(B, C)
    big = G.random_walks_device(5, 128, 3, start=(1 << 33) + 7).cpu().numpy()
    assert np.isfinite(big).all() and not np.array_equal(big, A[7:12])


def test_walk_properties(G):
    X = G.random_walks_device(2000, 256, 0).cpu().numpy().astype(np.float64)
    lag1 = np.mean([np.corrcoef(x[:-1], x[1:])[0, 1] for x in X[:200]])
    assert lag1 > 0.8
    steps = np.diff(X, axis=1)
    # increments of a z-normalised walk: zero-mean, symmetric
    assert abs(steps.mean()) < 1e-3 and abs(((steps - steps.mean()) ** 3).mean()) < 1e-3


def test_empty_and_bad_args(G):
    from paper_2212_13297_b200 import UsageError

    assert G.random_walks_device(0, 64, 1).shape == (0, 64)
    with pytest.raises(UsageError):
        G.random_walks_device(4, 2048, 1)
