"""Exact full-scan k-NN on the B200 (K-scan + K-select).

Drop-in for reference pscan.py (/root/reference/pkg/src/seriesearch/pscan.py):
``brute_force_knn`` (:23-30), ``pscan_query`` (:33-135), ``pscan`` (:138-149),
plus ``knn_batch``, which answers a whole query block in one launch.
``num_threads`` / ``chunk_series`` are accepted for signature compatibility
and have no effect (the scan is one device pass).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import device_f32, ptr, require_cuda, stream_handle
from .errors import DataFileError, UsageError
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


def _read_dataset(dataset_path: str, n: int):
    from .core import read_series_file

    return read_series_file(dataset_path, n)


def pscan_query(dataset_path: str, n: int, query, k: int, num_threads: int = 1,
                chunk_series: int = 16384) -> ResultSet:
    """Exact k-NN of one query over a raw dataset file (pscan.py:33-135)."""
    if num_threads < 1:
        raise UsageError("num_threads must be at least 1")
    q = np.ascontiguousarray(query, dtype=np.float32).reshape(-1)
    if q.size != n:
        raise UsageError(f"query length {q.size} != {n}")
    return brute_force_knn(_read_dataset(dataset_path, n), q, k)


def pscan(dataset_path: str, n: int, queries, k: int, num_threads: int = 1) -> list[ResultSet]:
    """A whole workload through one batched device scan (pscan.py:138-149)."""
    Q = np.atleast_2d(np.ascontiguousarray(queries, dtype=np.float32))
    if Q.shape[1] != n:
        raise UsageError(f"query length {Q.shape[1]} != {n}")
    d2, ids = knn_batch(_read_dataset(dataset_path, n), Q, k)
    d2 = d2.cpu().numpy()
    ids = ids.cpu().numpy()
    return [ResultSet.from_arrays(d2[i], ids[i]) for i in range(Q.shape[0])]
