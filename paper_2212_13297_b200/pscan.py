"""Exact full-scan k-NN on the B200 (K-scan + K-select).

Drop-in for reference pscan.py (/root/reference/pkg/src/seriesearch/pscan.py):
``brute_force_knn`` (:23-30), ``pscan_query`` (:33-135), ``pscan`` (:138-149),
plus ``knn_batch``, which answers a whole query block over resident rows in
one launch, and ``scan_file``, the streamed scan behind ``pscan_query`` /
``pscan`` (files larger than HBM; csrc/ingest.cu).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._device import device_f32, ptr, require_cuda, stream_handle
from .core import series_count
from .errors import UsageError
from .query import ResultSet

MAX_K = 256


def knn_batch(data, queries, k: int, id_base: int = 0):
    """Exact k-NN of every query row over ``data`` (both (rows, n) float32,
    numpy or torch).  Returns CUDA tensors (d2 (B,k) float32, ids (B,k) int64);
    missing answers are (+inf, -1)."""
    t = require_cuda()
    if k < 1:
        raise UsageError("k must be at least 1")
    if k > MAX_K:
        raise UsageError(f"k={k} exceeds the supported maximum {MAX_K}")
    X = device_f32(data)
    N, n = X.shape
    Q = device_f32(queries, n)
    B = Q.shape[0]
    d2 = t.empty((B, k), dtype=t.float32, device=X.device)
    ids = t.empty((B, k), dtype=t.int64, device=X.device)
    _lib.call("ssb_bruteforce_knn", ptr(X), N, n, ptr(Q), B, k, int(id_base), ptr(d2), ptr(ids),
              stream_handle())
    return d2, ids


def brute_force_knn(data, query, k: int) -> ResultSet:
    """Single-pass exact scan of one query (pscan.py:23-30)."""
    q = np.ascontiguousarray(query, dtype=np.float32).reshape(-1)
    d2, ids = knn_batch(data, q[None, :], k)
    d2 = d2.cpu().numpy()[0]
    ids = ids.cpu().numpy()[0]
    return ResultSet.from_arrays(d2, ids)


def scan_file(dataset_path: str, n: int, queries, k: int, first: int = 0, count: int | None = None, *,
              chunk_bytes: int = 256 << 20, threads: int = 0, stream=None):
    """Exact k-NN of a query block over rows [first, first + count) of a raw
    dataset FILE of any size, streamed through the device (``ssb_scan_file``):
    pinned double buffer -> copy stream -> K-scan against the running k-th key
    -> K-select -> merge, the read, copy and scan of consecutive chunks
    overlapped (the B200 form of pscan.py:50-135's reader thread, two-slot
    chunk buffer and shared best-so-far).  Neither HBM nor host memory holds
    the file.  Returns CUDA tensors (d2 (B,k), ids (B,k) = file row positions)
    and ``{"bytes", "seconds", "chunks", "GBps"}``."""
    t = require_cuda()
    if k < 1:
        raise UsageError("k must be at least 1")
    if k > MAX_K:
        raise UsageError(f"k={k} exceeds the supported maximum {MAX_K}")
    series_count(dataset_path, n)  # DataFileError / UsageError first, like the reference
    Q = device_f32(queries, n)
    B = Q.shape[0]
    d2 = t.empty((B, k), dtype=t.float32, device=Q.device)
    ids = t.empty((B, k), dtype=t.int64, device=Q.device)
    st = (ctypes.c_double * 3)()
    _lib.call("ssb_scan_file", dataset_path.encode(), int(first), -1 if count is None else int(count), int(n),
              ptr(Q), B, int(k), int(chunk_bytes), int(threads), ptr(d2), ptr(ids), stream_handle(stream), st)
    secs = st[1]
    return d2, ids, {"bytes": int(st[0]), "seconds": secs, "chunks": int(st[2]),
                     "GBps": (st[0] / secs / 1e9) if secs > 0 else None}


def _chunk_bytes(chunk_series: int, n: int) -> int:
    # the reference's chunk (rows per reader slot) as a lower bound; at least
    # 64 MB per device chunk so the per-chunk launches stay long
    return max(int(chunk_series) * 4 * n, 64 << 20)


def pscan_query(dataset_path: str, n: int, query, k: int, num_threads: int = 1,
                chunk_series: int = 16384) -> ResultSet:
    """Exact k-NN of one query over a raw dataset file (pscan.py:33-135),
    streamed: the file may be larger than HBM.  ``num_threads`` host threads
    read each chunk."""
    if num_threads < 1:
        raise UsageError("num_threads must be at least 1")
    if chunk_series < 1:
        raise UsageError("chunk_series must be at least 1")
    q = np.ascontiguousarray(query, dtype=np.float32).reshape(-1)
    series_count(dataset_path, n)
    if q.size != n:
        raise UsageError(f"query length {q.size} != {n}")
    d2, ids, _ = scan_file(dataset_path, n, q[None, :], k, chunk_bytes=_chunk_bytes(chunk_series, n),
                           threads=num_threads)
    return ResultSet.from_arrays(d2.cpu().numpy()[0], ids.cpu().numpy()[0])


def pscan(dataset_path: str, n: int, queries, k: int, num_threads: int = 1) -> list[ResultSet]:
    """A whole workload through one streamed pass over the file (pscan.py:138-149:
    the reference scans the file once per query; here every query shares each
    chunk's read, copy and scan)."""
    if num_threads < 1:
        raise UsageError("num_threads must be at least 1")
    Q = np.atleast_2d(np.ascontiguousarray(queries, dtype=np.float32))
    series_count(dataset_path, n)
    if Q.shape[1] != n:
        raise UsageError(f"query length {Q.shape[1]} != {n}")
    d2, ids, _ = scan_file(dataset_path, n, Q, k, threads=num_threads)
    d2 = d2.cpu().numpy()
    ids = ids.cpu().numpy()
    return [ResultSet.from_arrays(d2[i], ids[i]) for i in range(Q.shape[0])]
