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


@pytest.mark.parametrize("n,N,B,k", [(256, 100_003, 1, 100), (96, 30_001, 2, 10)])
def test_bruteforce_row_scan_direct_kernel(ssb, oracle, monkeypatch, n, N, B, k):
    """The direct-load row scan (the path of rows that are not 16-byte aligned;
    forced here by the A/B switch) and a misaligned view of the rows answer
    like the streamed kernel: the oracle's ids and d2 bits."""
    import torch
    X = random_walks(N, n, 3100 + N)
    Q = (X[[N // 3, N // 5][:B]] + np.float32(0.02)).astype(np.float32)
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    monkeypatch.setenv("SSB_ROWSCAN_DIRECT", "1")
    d2, ids = ssb.knn_batch(X, Q, k)
    monkeypatch.delenv("SSB_ROWSCAN_DIRECT")
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))
    # rows starting 4 bytes past a 16-byte boundary
    buf = torch.empty(N * n + 1, dtype=torch.float32, device="cuda")
    buf[1:].copy_(torch.from_numpy(X).reshape(-1))
    Xm = buf[1:].view(N, n)
    assert Xm.data_ptr() % 16 == 4
    d2, ids = ssb.knn_batch(Xm, Q, k)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


def test_bruteforce_row_scan_easy_and_hard_bounds(ssb, oracle):
    """The class-minimum bound of the streamed row scan: a query with many
    near-duplicates (the bound collapses at once: nearly every row abandoned
    after its first block), a far query (nothing abandoned early) and k larger
    than the rows of a range."""
    N, n = 200_000, 256
    X = random_walks(N, n, 4242)
    rng = np.random.default_rng(7)
    for i in range(300):                       # 300 near copies of row 1000 spread over the ranges
        X[(i * 661 + 17) % N] = X[1000] + np.float32(1e-3) * rng.standard_normal(n).astype(np.float32)
    near = X[[1000]].copy()
    far = (X[[5]] * np.float32(-3.0) + np.float32(2.0)).astype(np.float32)
    for Q, k in ((near, 100), (near, 256), (far, 100), (np.concatenate([near, far]), 1)):
        d2, ids = ssb.knn_batch(X, Q, k)
        od2, oid = oracle.knn_scan(X, Q, k, threads=8)
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


# ---------------------------------------------------------------------------
# streamed file scan (pscan.py:33-149 pscan_query / pscan; csrc/ingest.cu
# scan_file): chunks read, copied and scanned in a pipeline, the running k-th
# key carried from chunk to chunk.  Small chunk sizes force many chunks (and a
# ragged last one) so every bound hand-over is exercised.

def _write(tmp_path, X, name="data.bin"):
    p = tmp_path / name
    np.ascontiguousarray(X, np.float32).tofile(p)
    return str(p)


@pytest.mark.parametrize("n,N,B,k,chunk_rows", [(256, 50_003, 1, 10, 4096), (256, 50_003, 3, 100, 7000),
                                                (96, 40_001, 37, 10, 5000), (64, 30_000, 200, 1, 30_000),
                                                (128, 9_999, 5, 256, 1000), (256, 2_000, 1, 1, 333)])
def test_scan_file_matches_oracle(ssb, oracle, tmp_path, n, N, B, k, chunk_rows):
    X = random_walks(N, n, 5000 + N)
    Q = np.concatenate([random_walks(B - 1, n, 6000 + B), X[[N // 2]] + np.float32(0.01)]).astype(np.float32)
    path = _write(tmp_path, X)
    d2, ids, st = ssb.scan_file(path, n, Q, k, chunk_bytes=chunk_rows * 4 * n, threads=4)
    assert st["chunks"] == (N + chunk_rows - 1) // chunk_rows and st["bytes"] == X.nbytes
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))


def test_scan_file_ties_across_chunks(ssb, oracle, tmp_path):
    """Exact duplicates in different chunks: the lowest file position wins
    (pscan.py's answers equal the nested-loop scan's, ties to the lower id)."""
    X = random_walks(20_000, 256, 91)
    for i in (3, 7_777, 19_999):
        X[i] = X[12_345]
    path = _write(tmp_path, X)
    for B in (1, 9):  # row shape and dense shape
        Q = np.repeat(X[[12_345]], B, axis=0)
        d2, ids, _ = ssb.scan_file(path, 256, Q, 3, chunk_bytes=3000 * 1024)
        assert [list(r) for r in ids.cpu().numpy()] == [[3, 7_777, 12_345]] * B
        assert (d2.cpu().numpy() == 0).all()


def test_scan_file_subrange_edges_and_errors(ssb, oracle, tmp_path):
    X = random_walks(5_000, 64, 17)
    path = _write(tmp_path, X)
    Q = random_walks(6, 64, 18)
    # rows [1000, 3000): ids are file positions
    d2, ids, _ = ssb.scan_file(path, 64, Q, 5, first=1000, count=2000, chunk_bytes=700 * 256)
    od2, oid = oracle.knn_scan(X[1000:3000], Q, 5)
    assert np.array_equal(ids.cpu().numpy(), oid + 1000)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))
    # k > rows pads with (inf, -1); an empty range answers nothing
    d2, ids, _ = ssb.scan_file(path, 64, Q[:2], 8, first=4995, chunk_bytes=2 * 256)
    assert (ids.cpu().numpy()[:, 5:] == -1).all() and np.isinf(d2.cpu().numpy()[:, 5:]).all()
    d2, ids, _ = ssb.scan_file(path, 64, Q, 4, first=5000)
    assert (ids.cpu().numpy() == -1).all()
    with pytest.raises(ssb.DataFileError):
        ssb.scan_file(str(tmp_path / "missing.bin"), 64, Q, 1)
    with pytest.raises(ssb.UsageError):
        ssb.scan_file(path, 96, Q, 1)          # 5000 x 64 floats is not a whole number of 96-point series
    with pytest.raises(ssb.UsageError):
        ssb.scan_file(path, 64, Q, 1, first=4000, count=2000)
    with pytest.raises(ssb.UsageError):
        ssb.scan_file(path, 64, Q, 0)


def test_pscan_entry_points_stream_the_file(ssb, oracle, tmp_path):
    """pscan_query / pscan (pscan.py:33-149) through the streamed scan: the same
    ResultSets as the oracle, whatever chunk_series / num_threads say."""
    X = random_walks(30_000, 256, 23)
    path = _write(tmp_path, X)
    Q = random_walks(4, 256, 24)
    od2, oid = oracle.knn_scan(X, Q, 7)
    for t, cs in ((1, 16384), (4, 100), (16, 1 << 20)):
        rs = ssb.pscan_query(path, 256, Q[1], 7, num_threads=t, chunk_series=cs)
        assert [p for _, p in rs.entries()] == list(oid[1])
        assert rs.distances_sq() == [float(v) for v in od2[1]]
    rss = ssb.pscan(path, 256, Q, 7, num_threads=2)
    assert [[p for _, p in r.entries()] for r in rss] == [list(r) for r in oid]
    with pytest.raises(ssb.UsageError):
        ssb.pscan_query(path, 256, Q[0], 7, num_threads=0)
    with pytest.raises(ssb.UsageError):
        ssb.pscan_query(path, 256, Q[0][:100], 7)
