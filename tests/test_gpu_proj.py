"""K-proj, the projected lower-bound filter (csrc/proj.cu): a tensor-core
pass over the rows' d DCT-II coefficients under the approximate phase's
bounds, every emitted row rescored exactly.  Answers must be the oracle's
(pscan.py:23-30 brute_force_knn restated: ids identical, squared distances
bit-identical) whatever the bound's quality: easy queries (sigma = 0.01, 0.1)
are answered from their segments, hard ones (sigma = 1.0; or any query once
its segment is forced tiny) fall back to the full filter."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def walks():
    import paper_2212_13297_b200 as ssb
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(300_000, 256, 11)
    Qs = {s: G.noise_queries(X, 64, s, 12) for s in (0.01, 0.1, 1.0)}
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=3000))
    return ssb, X, Qs, idx, ssb.QueryEngine(idx)


def check(oracle, X, Q, k, d2, ids, what):
    od2, oid = oracle.knn_scan(X, Q, k, threads=THREADS)
    gids, gd2 = ids.cpu().numpy(), d2.cpu().numpy()
    bad = np.nonzero(~(np.all(gids == oid, axis=1) & np.all(bits(gd2) == bits(od2), axis=1)))[0]
    assert bad.size == 0, f"{what}: {bad.size} of {len(Q)} queries differ (first {bad[:5]})"


def test_projection_built_for_random_walks(walks):
    ssb, X, Qs, idx, eng = walks
    assert idx.info.proj_dim == 62
    assert idx.info.proj_energy > 0.95


@pytest.mark.parametrize("sigma", [0.01, 0.1, 1.0])
@pytest.mark.parametrize("k", [1, 10, 100])
def test_proj_route_exact(walks, oracle, sigma, k):
    ssb, X, Qs, idx, eng = walks
    Q = Qs[sigma]
    d2, ids, _, st = eng.knn_device(Q, k, route="proj", want_stats=True)
    check(oracle, X, Q, k, d2, ids, f"proj sigma={sigma} k={k}")
    routes = st[:, 7]
    assert set(np.unique(routes)) <= {1, 2}
    if sigma <= 0.1:
        assert (routes == 2).mean() > 0.9, routes  # the easy queries are settled by K-proj


def test_proj_segment_overflow_falls_back(walks, oracle, monkeypatch):
    ssb, X, Qs, idx, eng = walks
    monkeypatch.setenv("SSB_PROJ_SEG", "8")  # every query with more than 8 candidates overflows
    Q = Qs[0.1]
    for k in (1, 10):
        d2, ids, _, st = eng.knn_device(Q, k, route="proj", want_stats=True)
        check(oracle, X, Q, k, d2, ids, f"proj forced overflow k={k}")
    assert (st[:, 7] == 1).any()


def test_proj_auto_route_exact(walks, oracle):
    ssb, X, Qs, idx, eng = walks
    Q = np.concatenate([Qs[0.01], Qs[0.1], Qs[1.0]])
    for k in (1, 10):
        d2, ids, _ = eng.knn_device(Q, k, route="auto")
        check(oracle, X, Q, k, d2, ids, f"auto k={k}")


def test_no_projection_for_isotropic_rows(oracle):
    """I.i.d. Gaussian rows spread their energy evenly: 64 of 256 basis vectors
    hold ~25% of it, the bound would not prune, no operand is built, and route
    proj answers on the full filter."""
    import paper_2212_13297_b200 as ssb

    rng = np.random.default_rng(5)
    X = rng.standard_normal((50_000, 256)).astype(np.float32)
    Q = rng.standard_normal((32, 256)).astype(np.float32)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=2000))
    assert idx.info.proj_dim == 0
    eng = ssb.QueryEngine(idx)
    d2, ids, _ = eng.knn_device(Q, 10, route="proj")
    check(oracle, X, Q, 10, d2, ids, "isotropic proj")


def test_proj_index_round_trip(walks, oracle, tmp_path):
    """A written index, loaded back, rebuilds its projection operand (same
    answers)."""
    ssb, X, Qs, idx, eng = walks
    from paper_2212_13297_b200 import persist

    persist.write_index(idx, str(tmp_path / "ix"))
    idx2 = persist.load_index(str(tmp_path / "ix"))
    base = idx2.index if hasattr(idx2, "index") else idx2
    assert base.info.proj_dim == 62
    eng2 = ssb.QueryEngine(idx2)
    Q = Qs[0.1][:16]
    d2, ids, _ = eng2.knn_device(Q, 10, route="proj")
    check(oracle, X, Q, 10, d2, ids, "loaded index proj")
