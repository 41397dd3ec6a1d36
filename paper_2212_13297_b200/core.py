"""Host-side series primitives: coercion, z-normalisation and raw file I/O.

Mirrors reference core.py (/root/reference/pkg/src/seriesearch/core.py:1-159)
for the plumbing around the device path (the canonical distance itself,
``ed2_batch``, runs on the B200: pscan.py / csrc/scan.cu).
"""

from __future__ import annotations

import os

import numpy as np

from .errors import DataFileError, UsageError

DTYPE = np.dtype("<f4")
CONSTANT_SD = 1e-8


def as_series(values) -> np.ndarray:
    s = np.ascontiguousarray(values, dtype=DTYPE)
    if s.ndim != 1 or s.size == 0:
        raise UsageError("a series must be a non-empty 1-D vector")
    return s


def z_normalize(s) -> np.ndarray:
    """Mean 0 / population sd 1; constant series -> zeros (core.py:33-47)."""
    s = as_series(s)
    if not np.isfinite(s).all():
        raise UsageError("series contains non-finite values")
    x = s.astype(np.float64)
    mu = x.mean()
    sd = x.std()
    if sd < CONSTANT_SD:
        return np.zeros_like(s)
    return ((x - mu) / sd).astype(DTYPE)


def write_series_file(path: str, data: np.ndarray) -> int:
    arr = np.ascontiguousarray(data, dtype=DTYPE)
    try:
        with open(path, "wb") as f:
            f.write(arr.tobytes())
    except OSError as exc:
        raise DataFileError(f"{path}: {exc}") from exc
    return arr.nbytes


def series_count(path: str, n: int) -> int:
    try:
        size = os.path.getsize(path)
    except OSError as exc:
        raise DataFileError(f"{path}: {exc}") from exc
    if size % (4 * n) != 0:
        raise UsageError(f"{path}: size {size} is not a multiple of one {n}-point series")
    return size // (4 * n)


def read_series_file(path: str, n: int, count: int | None = None) -> np.ndarray:
    total = series_count(path, n)
    if count is None:
        count = total
    elif count > total:
        raise UsageError(f"{path}: requested {count} series, file has {total}")
    try:
        data = np.fromfile(path, dtype=DTYPE, count=count * n)
    except OSError as exc:
        raise DataFileError(f"{path}: {exc}") from exc
    return data.reshape(count, n)
