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


class QueryEngine:
    """Answers exact k-NN queries against one HBM-resident index.

    ``exact_knn`` keeps the reference signature (query.py:296-348) and
    returns ``(ResultSet, QueryStats)``; ``exact_knn_batch`` answers a whole
    block in one device pass (the only API addition); and
    ``knn_device`` is the zero-copy form for device-resident query blocks.
    ``lmax`` bounds the leaves the approximate phase visits and ``eapca_th``
    feeds the reference's routing rule (route="eapca"); ``sax_th`` and
    ``num_threads`` are validated and only select the reported phase label.
    The answers do not depend on any of them (the reference's path-invariance
    property, test_query.py:213-228).
    """

    def __init__(self, index):
        from .persist import QueryableIndex

        self.index = index
        self._si = index.index if isinstance(index, QueryableIndex) else index
        self.settings = self._si.settings
        self.total_leaves = int(self._si.info.num_leaves)
        self.total_series = int(self._si.info.dataset_size)

    def close(self) -> None:
        pass

    ROUTES = {"auto": 0, "tree": 1, "tensor": 2, "eapca": 3, "proj": 4}

    def knn_device(self, Q, k: int, want_stats: bool = False, eapca_th: float = 0.25,
                   route: str = "auto", lmax: int = 80):
        """(d2 (B,k) f32, ids (B,k) i64, pos (B,k) i64) CUDA tensors [+ stats (B,8) u32,
        the SSB_QUERY_STATS columns of include/seriesearch_b200.h].

        ``route``: "auto" picks, per query, the cheaper exact path by a
        B200-calibrated cost model; "eapca" applies the
        reference's eapca_th rule (weak envelope pruning -> dense scan path);
        "tree" / "tensor" force one path.  Answers are identical either way."""
        from . import _lib
        from ._device import device_f32, ptr, require_cuda, stream_handle

        t = require_cuda()
        if k < 1:
            raise UsageError("k must be at least 1")
        X = device_f32(Q, self.settings.series_length)
        B = X.shape[0]
        d2 = t.empty((B, k), dtype=t.float32, device=X.device)
        ids = t.empty((B, k), dtype=t.int64, device=X.device)
        pos = t.empty((B, k), dtype=t.int64, device=X.device)
        stats = np.zeros((B, _lib.QUERY_STATS), dtype=np.uint32) if want_stats else None
        if route not in self.ROUTES:
            raise UsageError(f"route must be one of {sorted(self.ROUTES)}")
        if lmax < 1:
            raise UsageError("lmax must be at least 1")
        cfg = _lib.QueryCfg(float(eapca_th), self.ROUTES[route], int(lmax))
        import ctypes as _ct

        _lib.call("ssb_query", self._si.handle, ptr(X), B, k, _ct.byref(cfg), ptr(d2), ptr(ids), ptr(pos),
                  stats.ctypes.data_as(_lib.P) if want_stats else None, stream_handle())
        return (d2, ids, pos, stats) if want_stats else (d2, ids, pos)

    def knn_device_multi(self, calls, eapca_th: float = 0.25, route: str = "auto", lmax: int = 80):
        """Several query blocks in one call: ``calls`` = [(Q, k), ...] ->
        [(d2, ids, pos), ...] CUDA tensors, each as ``knn_device(Q, k)``.
        The blocks are enqueued back to back with one host round trip for all
        of them (ssb_query_multi) instead of one per block."""
        import ctypes as _ct

        from . import _lib
        from ._device import device_f32, ptr, require_cuda, stream_handle

        t = require_cuda()
        if route not in self.ROUTES:
            raise UsageError(f"route must be one of {sorted(self.ROUTES)}")
        nc = len(calls)
        Xs, outs = [], []
        for Q, k in calls:
            if k < 1:
                raise UsageError("k must be at least 1")
            X = device_f32(Q, self.settings.series_length)
            B = X.shape[0]
            Xs.append(X)
            outs.append((t.empty((B, k), dtype=t.float32, device=X.device),
                         t.empty((B, k), dtype=t.int64, device=X.device),
                         t.empty((B, k), dtype=t.int64, device=X.device)))
        P = _ct.c_void_p * max(1, nc)
        I = _ct.c_int32 * max(1, nc)
        cfg = _lib.QueryCfg(float(eapca_th), self.ROUTES[route], int(lmax))
        _lib.call("ssb_query_multi", self._si.handle, nc, P(*[X.data_ptr() for X in Xs]),
                  I(*[X.shape[0] for X in Xs]), I(*[int(k) for _, k in calls]), _ct.byref(cfg),
                  P(*[o[0].data_ptr() for o in outs]), P(*[o[1].data_ptr() for o in outs]),
                  P(*[o[2].data_ptr() for o in outs]), stream_handle())
        return outs

    def exact_knn_arrays(self, queries, k: int, eapca_th: float = 0.25):
        """Batched public form over HOST buffers: (d2, ids, pos) numpy arrays
        (B, k); the H2D copy of the queries and the D2H copy of the answers
        are part of the call."""
        d2, ids, pos = self.knn_device(queries, k, eapca_th=eapca_th)
        return d2.cpu().numpy(), ids.cpu().numpy(), pos.cpu().numpy()

    def _stats(self, row, cfg: QueryConfig, wall: float) -> QueryStats:
        """QueryStats (query.py:102-114) from one row of the device counters.

        ``series_read`` counts the series whose raw values the query actually
        read (the reference's SeriesStore accounting, persist.py:88-122): on the
        index route the approximate phase's exactly scanned series plus the
        LB_SAX survivors (an early-abandoned survivor was read in part); on the
        tensor-core route every row (its BF16 copy streams through the filter)."""
        n = self.settings.series_length
        cand_leaves, cand_series, seed_rows = int(row[0]), int(row[1]), int(row[2])
        seed_leaves, words, tc = int(row[4]), int(row[5]), int(row[7])
        st = QueryStats()
        st.visited_leaves = seed_leaves
        st.candidate_leaves = cand_leaves
        st.candidate_series = cand_series
        st.eapca_pr = 1.0 - cand_leaves / max(1, self.total_leaves)
        st.sax_pr = 1.0 - cand_series / max(1, self.total_series)
        # phase label by the reference's decision rules (query.py:321-341)
        if tc or st.eapca_pr < cfg.eapca_th:
            st.phase_reached = "scan2"
        elif st.sax_pr < cfg.sax_th:
            st.phase_reached = "scan3"
        elif cand_series:
            st.phase_reached = "4"
        elif cand_leaves:
            st.phase_reached = "3"
        else:
            st.phase_reached = "1"
        if tc:
            # a pass over every row's BF16 operand (route 2, K-proj: its d projection
            # coefficients; route 1: the whole row) + the exact rescoring
            width = int(self._si.info.proj_dim) if tc == 2 else n
            st.series_read = self.total_series
            st.bytes_read = self.total_series * width * 2 + cand_series * n * 4
        else:
            st.series_read = min(self.total_series, seed_rows + cand_series)
            st.bytes_read = st.series_read * n * 4 + words * 16  # rows + SAX words tested
        st.fraction_data_accessed = st.series_read / max(1, self.total_series)
        st.wall_seconds = wall
        return st

    def exact_knn_batch(self, queries, cfg: QueryConfig, route: str = "auto"):
        import time

        cfg.validate()
        Q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
        n = self.settings.series_length
        if Q.shape[1] != n:
            raise UsageError(f"query length {Q.shape[1]} does not match index series length {n}")
        if not np.isfinite(Q).all():
            raise UsageError("queries must be finite (documented deviation: NaN keys break ordering)")
        t0 = time.perf_counter()
        d2, ids, pos, stats = self.knn_device(Q, cfg.k, want_stats=True, eapca_th=cfg.eapca_th, lmax=cfg.lmax,
                                              route=route)
        d2, ids, pos = d2.cpu().numpy(), ids.cpu().numpy(), pos.cpu().numpy()
        wall = (time.perf_counter() - t0) / max(1, Q.shape[0])
        return [(ResultSet.from_arrays(d2[i], pos[i], ids[i]), self._stats(stats[i], cfg, wall))
                for i in range(Q.shape[0])]

    def exact_knn(self, query, cfg: QueryConfig):
        q = np.ascontiguousarray(query, dtype=np.float32)
        n = self.settings.series_length
        if q.ndim != 1 or q.size != n:
            raise UsageError(f"query length {q.size} does not match index series length {n}")
        return self.exact_knn_batch(q[None, :], cfg)[0]


def exact_knn(query, index, cfg: QueryConfig):
    """One-shot convenience wrapper (query.py:351-357)."""
    engine = QueryEngine(index)
    try:
        return engine.exact_knn(query, cfg)
    finally:
        engine.close()
