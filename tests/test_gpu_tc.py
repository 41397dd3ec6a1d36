"""K-tc: tcgen05/TMEM/TMA tensor-core filter.  The raw dot products must match
a BF16 matmul; the tensor-core query path must give answers identical to the
oracle (the filter only selects rows for exact float32 rescoring)."""

import ctypes

import numpy as np
import pytest

from conftest import random_walks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ssb():
    import paper_2212_13297_b200 as ssb

    return ssb


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# the tile-major pre-swizzled operand: 64-column K-chunks (SWIZZLE_128B) where
# n % 64 == 0, else 32-column chunks (SWIZZLE_64B): n = 96, 160, 224, 32
@pytest.mark.parametrize("n,B,N", [(256, 200, 1000), (96, 130, 777), (64, 5, 300), (128, 128, 128),
                                   (160, 70, 500), (224, 130, 400), (32, 40, 300)])
def test_tc_dot_matches_fp16_matmul(ssb, n, B, N):
    """The tcgen05 dot products of the FP16 operands (the filters' operand
    format) against a float64 matmul of the same FP16-rounded values."""
    import torch

    from paper_2212_13297_b200 import _lib

    Q = torch.from_numpy(random_walks(B, n, 1)).cuda()
    X = torch.from_numpy(random_walks(N, n, 2)).cuda()
    S = torch.full((B, N), float("nan"), dtype=torch.float32, device="cuda")
    _lib.call("ssb_tc_dot_debug", ctypes.c_void_p(Q.data_ptr()), B, ctypes.c_void_p(X.data_ptr()), N, n,
              ctypes.c_void_p(S.data_ptr()), None)
    ref = Q.half().double() @ X.half().double().T
    err = (S.double() - ref).abs().max().item()
    assert np.isfinite(S.cpu().numpy()).all()
    assert err < 1e-3, err


@pytest.mark.parametrize("k", [1, 10, 50])
def test_tensor_route_equals_oracle(ssb, oracle, k):
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(20_000, 256, 0, workers=4)
    s = ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=1000)
    idx = ssb.build_index_array(X, s)
    Q = np.concatenate([G.noise_queries(X, 40, 1.0, 1), G.noise_queries(X, 20, 0.1, 2),
                        random_walks(10, 256, 3)])
    d2, ids, _, st = ssb.QueryEngine(idx).knn_device(Q, k, want_stats=True, route="tensor")
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


def test_auto_route_mixed_block(ssb, oracle):
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(30_000, 256, 0, workers=4)
    s = ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=1000)
    idx = ssb.build_index_array(X, s)
    Q = np.concatenate([G.noise_queries(X, 50, 1.0, 1), G.noise_queries(X, 50, 0.01, 1)])
    eng = ssb.QueryEngine(idx)
    for k in (1, 10):
        d2, ids, _ = eng.knn_device(Q, k)
        od2, oid = oracle.knn_scan(X, Q, k, threads=8)
        assert np.array_equal(ids.cpu().numpy(), oid)
        assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))
        t2, tid, _ = eng.knn_device(Q, k, route="tree")
        assert np.array_equal(tid.cpu().numpy(), oid)


def test_tensor_route_ties(ssb, oracle):
    X = random_walks(5000, 128, 7)
    X[4000] = X[17]
    X[4999] = X[17]
    s = ssb.IndexSettings(series_length=128, dataset_size=len(X), leaf_threshold=300)
    idx = ssb.build_index_array(X, s)
    d2, ids, _ = ssb.QueryEngine(idx).knn_device(X[[17]], 3, route="tensor")
    assert list(ids.cpu().numpy()[0]) == [17, 4000, 4999]


@pytest.mark.parametrize("route", ["auto", "eapca", "tree", "tensor"])
def test_every_route_is_exact(ssb, oracle, route):
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(12_000, 256, 0, workers=4)
    s = ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=500)
    idx = ssb.build_index_array(X, s)
    Q = np.concatenate([G.noise_queries(X, 30, 1.0, 1), G.noise_queries(X, 30, 0.01, 1)])
    for k in (1, 5, 40):
        d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, k, route=route)
        od2, oid = oracle.knn_scan(X, Q, k, threads=8)
        assert np.array_equal(ids.cpu().numpy(), oid), (route, k)
        assert np.array_equal(bits(d2.cpu().numpy()), bits(od2)), (route, k)


@pytest.mark.parametrize("N,k", [(70, 100), (70, 20), (200, 100), (130, 1)])
def test_tensor_route_small_and_ragged(ssb, oracle, N, k):
    """Tiles past N are zero-filled by TMA; they must never become candidates
    (k > N keeps the bound at +inf)."""
    X = random_walks(N, 64, 9)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=64, dataset_size=N, leaf_threshold=4))
    Q = random_walks(3, 64, 10)
    od2, oid = oracle.knn_scan(X, Q, k)
    d2, ids, _, st = ssb.QueryEngine(idx).knn_device(Q, k, want_stats=True, route="tensor")
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert (st[:, 1] <= N).all()


@pytest.mark.parametrize("k", [33, 100, 300])
def test_tensor_route_large_k_buckets(ssb, oracle, k):
    """k > 32: no per-thread list, only the pooled bucket bound; 300 queries
    span three query blocks (one padded)."""
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(20_000, 128, 4, workers=4)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=128, dataset_size=len(X), leaf_threshold=800))
    Q = np.concatenate([G.noise_queries(X, 200, 0.1, 5), random_walks(100, 128, 6)])
    d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, k, route="tensor")
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


@pytest.mark.parametrize("N,k", [(300, 32), (1000, 31), (2000, 2), (517, 17)])
def test_tensor_route_warmup_revisits(ssb, oracle, N, k):
    """Few tiles per CTA: the warm-up tiles are rescanned; their rows must not
    enter a thread's own top-k list twice."""
    X = random_walks(N, 96, 11)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=96, dataset_size=N, leaf_threshold=50))
    Q = np.concatenate([X[:5] + 0.01, random_walks(60, 96, 12)]).astype(np.float32)
    d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, k, route="tensor")
    od2, oid = oracle.knn_scan(X, Q, k)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


@pytest.mark.parametrize("hook,value", [("SSB_TEST_TC_CAP", "300"), ("SSB_TEST_TC_CAP", "1"),
                                        ("SSB_TEST_SELECT_CAP", "12")])
def test_tensor_route_overflow_paths(ssb, oracle, monkeypatch, hook, value):
    """Candidate-buffer overflow: retried with the filter's final bounds, then
    (still overflowing) answered on the general path; a select overflow goes
    to the general path too.  Answers stay exact."""
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(8000, 256, 13, workers=4)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=400))
    Q = np.concatenate([G.noise_queries(X, 30, 1.0, 14), G.noise_queries(X, 10, 0.01, 15)])
    monkeypatch.setenv(hook, value)
    for k in (1, 10):
        d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, k, route="tensor")
        od2, oid = oracle.knn_scan(X, Q, k, threads=8)
        assert np.array_equal(ids.cpu().numpy(), oid), (hook, value, k)
        assert np.array_equal(bits(d2.cpu().numpy()), bits(od2)), (hook, value, k)


@pytest.mark.parametrize("route", ["auto", "tensor", "tree"])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_non_finite_queries_rejected(ssb, route, bad):
    X = random_walks(3000, 64, 21)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=64, dataset_size=len(X), leaf_threshold=100))
    Q = random_walks(5, 64, 22)
    Q[3, 17] = bad
    with pytest.raises(ssb.UsageError):
        ssb.QueryEngine(idx).knn_device(Q, 3, route=route)


@pytest.mark.parametrize("route", ["auto", "tree"])
def test_query_multi_equals_separate_calls(ssb, oracle, route):
    """ssb_query_multi: blocks with different k (and an empty one) enqueued
    together answer exactly like one call per block (lean tensor-core path for
    route auto, the general path for route tree)."""
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(20_000, 256, 4, workers=4)
    s = ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=1000)
    eng = ssb.QueryEngine(ssb.build_index_array(X, s))
    Q1 = G.noise_queries(X, 50, 0.1, 5)
    Q2 = G.noise_queries(X, 70, 1.0, 6)
    calls = [(Q1, 1), (Q2, 10), (Q1[:0], 3), (Q2[:9], 100)]
    outs = eng.knn_device_multi(calls, route=route)
    for (Q, k), (d2, ids, pos) in zip(calls, outs):
        assert d2.shape == (len(Q), k)
        if len(Q) == 0:
            continue
        od2, oid = oracle.knn_scan(X, Q, k, threads=8)
        assert np.array_equal(ids.cpu().numpy(), oid)
        assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))
        e2, eid, epos = eng.knn_device(Q, k, route=route)
        assert np.array_equal(pos.cpu().numpy(), epos.cpu().numpy())


def test_query_multi_overflow_retry(ssb, oracle, monkeypatch):
    """A candidate-buffer overflow inside a multi call is retried per block."""
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(8000, 128, 8, workers=2)
    s = ssb.IndexSettings(series_length=128, dataset_size=len(X), leaf_threshold=500)
    eng = ssb.QueryEngine(ssb.build_index_array(X, s))
    Q = G.noise_queries(X, 40, 1.0, 9)
    monkeypatch.setenv("SSB_TEST_TC_CAP", "64")
    outs = eng.knn_device_multi([(Q, 5), (Q[:7], 1)], route="tensor")
    for (Qc, k), (d2, ids, _) in zip([(Q, 5), (Q[:7], 1)], outs):
        od2, oid = oracle.knn_scan(X, Qc, k, threads=8)
        assert np.array_equal(ids.cpu().numpy(), oid)
        assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))
