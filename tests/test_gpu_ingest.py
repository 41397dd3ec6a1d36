"""Ingest pipeline (csrc/ingest.cu): file -> pinned double buffer -> HBM.
Rows must arrive bit-identical to np.fromfile (core.py:113-159 read_series_file),
across chunk boundaries, ragged tails, shards and thread counts; a build from
the file equals the build from the same array."""

import numpy as np
import pytest

from conftest import random_walks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ssb():
    import paper_2212_13297_b200 as ssb

    return ssb


@pytest.fixture(scope="module")
def data_file(tmp_path_factory):
    X = random_walks(10_007, 64, 41)
    p = tmp_path_factory.mktemp("ingest") / "d.bin"
    X.tofile(p)
    return str(p), X


@pytest.mark.parametrize("chunk_rows,threads", [(1000, 1), (777, 3), (1 << 20, 0), (1, 2)])
def test_ingest_equals_fromfile(ssb, data_file, chunk_rows, threads):
    path, X = data_file
    D, st = ssb.ingest_file(path, 64, chunk_bytes=chunk_rows * 256, threads=threads)
    assert D.shape == X.shape and D.is_cuda
    assert np.array_equal(D.cpu().numpy().view(np.uint32), X.view(np.uint32))
    assert st["bytes"] == X.nbytes


@pytest.mark.parametrize("first,count", [(0, 1), (1234, 5000), (10_006, 1), (9_000, None), (5, 0)])
def test_ingest_shard(ssb, data_file, first, count):
    path, X = data_file
    D, _ = ssb.ingest_file(path, 64, first, count, chunk_bytes=999 * 256)
    hi = len(X) if count is None else first + count
    assert np.array_equal(D.cpu().numpy(), X[first:hi])


def test_ingest_errors(ssb, data_file, tmp_path):
    path, X = data_file
    with pytest.raises(ssb.DataFileError):
        ssb.ingest_file(str(tmp_path / "missing.bin"), 64)
    with pytest.raises(ssb.UsageError):
        ssb.ingest_file(path, 48)  # 10007 x 64 floats is not a whole number of 48-point series
    with pytest.raises(ssb.UsageError):
        ssb.ingest_file(path, 64, 10_000, 8)


def test_build_from_file_equals_build_from_array(ssb, data_file, oracle):
    path, X = data_file
    s = ssb.IndexSettings(series_length=64, dataset_size=len(X), leaf_threshold=300)
    trace = ssb.BuildTrace()
    a = ssb.build_index(path, s, num_threads=4, trace=trace)
    b = ssb.build_index_array(X, s)
    assert trace.of_kind("ingest")[0][2]["bytes"] == X.nbytes
    ra, wa, oa = a.host_arrays()
    rb, wb, ob = b.host_arrays()
    assert np.array_equal(oa, ob) and np.array_equal(wa, wb) and np.array_equal(ra, rb)
    Q = X[:7] + np.float32(0.05)
    from paper_2212_13297_b200 import QueryEngine

    d2, ids = QueryEngine(a).knn_device(Q, 5)[:2]
    od2, oid = oracle.knn_scan(X, Q, 5)
    assert np.array_equal(ids.cpu().numpy(), oid)
