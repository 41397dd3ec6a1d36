"""Exact k-NN answering: configuration, result and statistics types.

Mirrors reference query.py (/root/reference/pkg/src/seriesearch/query.py):
``QueryConfig`` (:42-58), ``ResultSet`` (:61-99), ``QueryStats`` (:102-114).
The engine itself (``QueryEngine``) drives the B200 kernels; see engine.py.

Ordering deviation (documented in DESIGN.md): answers are ordered by
(squared distance, original series index), so ties resolve to the lowest
index exactly like pscan.py:23-30 ``brute_force_knn``, instead of the
reference engine's "earliest found" rule, which depends on visiting order.
"""

from __future__ import annotations

import bisect
import threading
from dataclasses import dataclass

import numpy as np

from .errors import UsageError


@dataclass
class QueryConfig:
    k: int = 1
    lmax: int = 80
    eapca_th: float = 0.25
    sax_th: float = 0.50
    num_threads: int = 1

    def validate(self) -> None:
        if self.k < 1:
            raise UsageError("k must be at least 1")
        if self.lmax < 1:
            raise UsageError("lmax must be at least 1")
        if not (0.0 <= self.eapca_th <= 1.0 and 0.0 <= self.sax_th <= 1.0):
            raise UsageError("thresholds must lie in [0, 1]")
        if self.num_threads < 1:
            raise UsageError("num_threads must be at least 1")


class ResultSet:
    """The k best answers: (squared distance, position), sorted.

    ``bsf`` is the k-th best squared distance.  ``insert`` keeps the
    reference's host-side semantics (query.py:77-89) for callers that fill a
    set by hand; sets produced by the engine come from ``from_arrays``.
    ``ids()`` additionally reports original series indices.
    """

    def __init__(self, k: int):
        self.k = k
        self._dists = [np.inf] * k
        self._positions: list[int | None] = [None] * k
        self._ids: list[int | None] = [None] * k
        self._lock = threading.Lock()
        self.bsf = np.inf

    @classmethod
    def from_arrays(cls, d2, positions, ids=None) -> "ResultSet":
        k = len(d2)
        rs = cls(k)
        rs._dists = [float(v) for v in d2]
        rs._positions = [None if int(p) < 0 else int(p) for p in positions]
        src = positions if ids is None else ids
        rs._ids = [None if int(p) < 0 else int(p) for p in src]
        rs.bsf = rs._dists[-1] if k else np.inf
        return rs

    def insert(self, dist: float, pos: int) -> bool:
        if dist >= self.bsf:
            return False
        with self._lock:
            if dist >= self._dists[-1]:
                return False
            at = bisect.bisect_right(self._dists, dist)
            self._dists.insert(at, dist)
            self._positions.insert(at, pos)
            self._ids.insert(at, pos)
            self._dists.pop()
            self._positions.pop()
            self._ids.pop()
            self.bsf = self._dists[-1]
            return True

    def distances_sq(self) -> list[float]:
        return list(self._dists)

    def positions(self) -> list[int | None]:
        return list(self._positions)

    def ids(self) -> list[int | None]:
        return list(self._ids)

    def entries(self) -> list[tuple[float, int | None]]:
        """(reported distance, position) pairs; sqrt happens here (query.py:94-99)."""
        return [
            (float(np.sqrt(d)) if np.isfinite(d) else float("inf"), p)
            for d, p in zip(self._dists, self._positions)
        ]


@dataclass
class QueryStats:
    phase_reached: str = "1"
    eapca_pr: float = 0.0
    sax_pr: float = 0.0
    visited_leaves: int = 0
    series_read: int = 0
    bytes_read: int = 0
    fraction_data_accessed: float = 0.0
    input_seconds: float = 0.0
    wall_seconds: float = 0.0
    candidate_leaves: int = 0
    candidate_series: int = 0
