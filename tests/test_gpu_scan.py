"""K-scan / K-select / K-sum parity on the B200 against the oracle and the
reference-generated golden vectors.  Bar: bit-exact (distances are compared
as float32 bit patterns, ids exactly)."""

import numpy as np
import pytest

from conftest import golden, random_walks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ssb():
    import paper_2212_13297_b200 as ssb

    return ssb


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("k", [1, 10, 100])
def test_bruteforce_matches_reference_golden(ssb, k):
    g = golden("knn")
    d2, ids = ssb.knn_batch(g["X"], g["Q"], k)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(g[f"d2_k{k}"]))
    assert np.array_equal(ids.cpu().numpy(), g[f"id_k{k}"])


def test_bruteforce_ties_lowest_index(ssb):
    g = golden("knn")
    _, ids = ssb.knn_batch(g["X"], g["Q"], 3)
    ids = ids.cpu().numpy()
    assert list(ids[6]) == [10, 2500, 2999]
    assert list(ids[7][:2]) == [1100, 1200]


@pytest.mark.parametrize("n", [16, 64, 96, 256, 320])
def test_every_distance_bitwise_equals_ed2_batch(ssb, n):
    g = golden("ed2")
    X, q = g[f"X{n}"], g[f"q{n}"]
    if n not in (64, 96, 128, 256):
        with pytest.raises(ssb.UsageError):
            ssb.knn_batch(X, q[None], 1)
        return
    d2, ids = ssb.knn_batch(X, q[None], X.shape[0])
    d2, ids = d2.cpu().numpy()[0], ids.cpu().numpy()[0]
    assert sorted(ids) == list(range(X.shape[0]))
    assert np.array_equal(bits(d2), bits(g[f"d2_{n}"][ids]))


@pytest.mark.parametrize("n,N,B,k", [(256, 20_011, 37, 10), (96, 9_999, 70, 7),
                                     (64, 5_000, 3, 100), (256, 1_000, 1, 256),
                                     (128, 333, 33, 1)])
def test_bruteforce_matches_oracle(ssb, oracle, n, N, B, k):
    X = random_walks(N, n, 1000 + N)
    Q = random_walks(B, n, 2000 + B)
    d2, ids = ssb.knn_batch(X, Q, k)
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


def test_bruteforce_edges(ssb, oracle):
    X = random_walks(5, 64, 1)
    d2, ids = ssb.knn_batch(X, X[:2], 8)          # k > N pads with (inf, -1)
    ids = ids.cpu().numpy()
    assert list(ids[0][:1]) == [0] and list(ids[0][5:]) == [-1, -1, -1]
    assert np.isinf(d2.cpu().numpy()[0][5:]).all()
    empty = np.zeros((0, 64), np.float32)
    d2, ids = ssb.knn_batch(empty, X[:1], 2)      # empty dataset
    assert (ids.cpu().numpy() == -1).all()
    d2, ids = ssb.knn_batch(X, np.zeros((0, 64), np.float32), 2)  # no queries
    assert d2.shape == (0, 2)
    with pytest.raises(ssb.UsageError):
        ssb.knn_batch(X, X[:1], 0)
    with pytest.raises(ssb.UsageError):
        ssb.knn_batch(X, X[:1, :32], 1)
    # id_base offsets ids (shard mode)
    _, ids = ssb.knn_batch(X, X[:1], 1, id_base=1000)
    assert int(ids.cpu().numpy()[0, 0]) == 1000


def test_brute_force_knn_resultset(ssb, oracle):
    X = random_walks(3000, 256, 5)
    q = random_walks(1, 256, 6)[0]
    rs = ssb.brute_force_knn(X, q, 5)
    od2, oid = oracle.knn_scan(X, q[None], 5)
    assert rs.distances_sq() == [float(v) for v in od2[0]]
    assert [p for _, p in rs.entries()] == list(oid[0])


def test_words_match_golden(ssb):
    from paper_2212_13297_b200.summarize import paa_words

    g = golden("words")
    for n in (96, 256):
        w, p = paa_words(g[f"X{n}"], with_paa=True)
        assert np.array_equal(bits(p.cpu().numpy()), bits(g[f"paa{n}"])), n
        assert np.array_equal(w.cpu().numpy(), g[f"words{n}"]), n


def test_words_match_oracle_large(ssb, oracle):
    from paper_2212_13297_b200.summarize import paa_words

    X = random_walks(50_000, 256, 9)
    bp = oracle.normal_breakpoints(256)
    assert np.array_equal(paa_words(X).cpu().numpy(), oracle.words(X, bp))


def test_segment_stats_match_golden(ssb):
    from paper_2212_13297_b200.summarize import segment_stats_matrix

    g = golden("stats")
    for name in ("root", "three", "fine", "width1"):
        mean, sd = segment_stats_matrix(g["X"], g[f"starts_{name}"], g[f"ends_{name}"])
        assert np.array_equal(bits(mean.cpu().numpy()), bits(g[f"mean_{name}"])), name
        assert np.array_equal(bits(sd.cpu().numpy()), bits(g[f"sd_{name}"])), name


@pytest.mark.parametrize("starts,ends", [([5, 20], [20, 31]),  # contiguous, not from 0
                                         ([0, 10, 3], [64, 40, 9]),  # overlapping / unsorted
                                         ([1, 63], [2, 64])])  # gaps
def test_segment_stats_general_segments(ssb, oracle, starts, ends):
    from paper_2212_13297_b200.summarize import segment_stats_matrix

    X = random_walks(3000, 64, 31)
    mean, sd = segment_stats_matrix(X, np.array(starts), np.array(ends))
    omean, osd = oracle.segment_stats(X, np.array(starts), np.array(ends))
    assert np.array_equal(bits(mean.cpu().numpy()), bits(omean))
    assert np.array_equal(bits(sd.cpu().numpy()), bits(osd))


@pytest.mark.parametrize("m,N", [(16, 1037), (32, 129), (33, 300), (64, 1), (1, 128), (7, 3001)])
def test_segment_stats_contiguous_partitions(ssb, oracle, m, N):
    """Contiguous partitions of [0, n): m <= 32 takes the shared-memory staged
    output path (coalesced block stores), larger m the direct stores; ragged
    last CTA included."""
    from paper_2212_13297_b200.summarize import segment_stats_matrix

    n = 256
    X = random_walks(N, n, 37 + m)
    cuts = np.linspace(0, n, m + 1).astype(np.int64)
    starts, ends = cuts[:-1], cuts[1:]
    mean, sd = segment_stats_matrix(X, starts, ends)
    omean, osd = oracle.segment_stats(X, starts, ends)
    assert np.array_equal(bits(mean.cpu().numpy()), bits(omean))
    assert np.array_equal(bits(sd.cpu().numpy()), bits(osd))


@pytest.mark.parametrize("starts,ends", [([0, 1000, 1500], [1500, 2048, 1501]),  # widths 1500, 1048, 1
                                         ([0], [2048])])                          # one 2048-wide segment
def test_segment_stats_wide_segments(ssb, oracle, starts, ends):
    """Segments wider than the reciprocal table (w > 1024, n = 2048): the
    division falls back to IEEE division and stays bit-identical to
    summarize.py:79-82."""
    from paper_2212_13297_b200.summarize import segment_stats_matrix

    X = random_walks(700, 2048, 41)
    mean, sd = segment_stats_matrix(X, np.array(starts), np.array(ends))
    omean, osd = oracle.segment_stats(X, np.array(starts), np.array(ends))
    assert np.array_equal(bits(mean.cpu().numpy()), bits(omean))
    assert np.array_equal(bits(sd.cpu().numpy()), bits(osd))


@pytest.mark.parametrize("n,N,B,k", [(256, 300_007, 1, 1), (256, 300_007, 1, 100), (96, 120_001, 2, 10),
                                     (64, 50_000, 4, 256), (128, 1_000, 3, 7), (256, 37, 1, 50)])
def test_bruteforce_few_queries_row_scan(ssb, oracle, n, N, B, k):
    """B <= 4: the row-parallel early-abandoning scan (every group on its own
    rows, bounds shared across groups and CTAs) -- ids and d2 bits equal the
    oracle; N < k pads with (inf, -1)."""
    X = random_walks(N, n, 3000 + N)
    Q = np.concatenate([random_walks(B - 1, n, 4000 + B), X[[N // 2]]]) if B > 1 else X[[N // 3]] + 0.01
    d2, ids = ssb.knn_batch(X, Q.astype(np.float32), k)
    od2, oid = oracle.knn_scan(X, Q.astype(np.float32), k, threads=8)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


def test_bruteforce_row_scan_ties(ssb, oracle):
    X = random_walks(70_000, 256, 77)
    for i in (5, 33_333, 69_999):
        X[i] = X[40_000]           # exact duplicates across CTAs and groups
    Q = X[[40_000]].copy()
    d2, ids = ssb.knn_batch(X, Q, 3)
    assert list(ids.cpu().numpy()[0]) == [5, 33_333, 40_000]
    od2, oid = oracle.knn_scan(X, Q, 10)
    d2, ids = ssb.knn_batch(X, Q, 10)
    assert np.array_equal(ids.cpu().numpy(), oid)
