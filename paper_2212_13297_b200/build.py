"""Index construction on the B200.

Drop-in for reference build.py (/root/reference/pkg/src/seriesearch/build.py):
``build_index`` (:363-458) keeps its signature and validation
(:380-403); ``SeriesIndex`` (:117-171) and ``BuildTrace`` (:70-82) keep their
names.  The work itself is the level-synchronous device build in
csrc/build.cu: every node above the leaf threshold is split
with the reference's own policy choice (tree.py:240-336), evaluated over all
of its members, and the members are stably partitioned into leaf-contiguous
HBM arrays.  The reference's threaded insertion, DBuffer/HBuffer/SBuffer and
flush protocol (build.py:32-211, 266-465) have no counterpart: leaves live in
HBM.  ``buffer_bytes``, ``dbsize``, ``flush_threshold`` and ``scratch_dir``
are validated like the reference and otherwise unused.
"""

from __future__ import annotations

import ctypes
import math
import threading

import numpy as np

from . import _lib
from ._device import device_f32, ptr, require_cuda, stream_handle
from .core import series_count
from .errors import UsageError
from .summarize import device_breakpoints
from .tree import Node, tree_from_records

DEFAULT_DBSIZE = 120_000
DBSIZE_SCALE_POINT = 1_000_000


def default_dbsize(dataset_size: int) -> int:
    """build.py:37-41 (validation only; there is no read chunking on the device)."""
    if dataset_size >= DBSIZE_SCALE_POINT:
        return DEFAULT_DBSIZE
    return max(1, math.ceil(DEFAULT_DBSIZE * dataset_size / DBSIZE_SCALE_POINT))


class BuildTrace:
    """Event recorder (build.py:70-82).  The device build notes one
    ``level`` event per level and one ``done`` event."""

    def __init__(self):
        self.events: list[tuple] = []
        self._lock = threading.Lock()

    def note(self, worker_id: int, kind: str, **info):
        with self._lock:
            self.events.append((worker_id, kind, info))

    def of_kind(self, kind: str):
        return [e for e in self.events if e[1] == kind]


class _Handle:
    """Owns one ssb_index* (freed with the last reference)."""

    def __init__(self, raw: ctypes.c_void_p):
        self.raw = raw

    def __del__(self):
        if self.raw:
            try:
                _lib.load().ssb_index_free(self.raw)
            except Exception:  # pragma: no cover - interpreter teardown
                pass
            self.raw = None


class SeriesIndex:
    """The built index: an HBM-resident tree shard plus its host-side view."""

    def __init__(self, settings, handle: _Handle, trace: BuildTrace | None = None):
        self.settings = settings
        self._handle = handle
        self.trace = trace
        info = _lib.IndexInfo()
        _lib.call("ssb_index_info", handle.raw, ctypes.byref(info))
        self.info = info
        self._root: Node | None = None
        self.id_base = int(info.id_base)

    @property
    def root(self) -> Node:
        """Host view of the tree (tree.py Node graph), materialised on first use:
        the device index does not need it to answer queries."""
        if self._root is None:
            recs = []
            for i in range(self.info.num_nodes):
                r = _lib.NodeRec()
                _lib.call("ssb_index_node", self._handle.raw, i, ctypes.byref(r))
                recs.append(r)
            self._root = tree_from_records(recs)
        return self._root

    @property
    def handle(self):
        return self._handle.raw

    def leaves_inorder(self) -> list[Node]:
        return list(self.root.iter_leaves())

    def device_arrays(self):
        """(X, words, orig, inv) raw device pointers, leaf order."""
        X, W, O, I = (ctypes.c_void_p() for _ in range(4))
        _lib.call("ssb_index_arrays", self.handle, ctypes.byref(X), ctypes.byref(W), ctypes.byref(O),
                  ctypes.byref(I))
        return X.value, W.value, O.value, I.value

    def host_arrays(self):
        """Leaf-ordered rows (N, n) float32, words (N, 16) uint8 and the
        original index of every position (N,) int64, copied to the host."""
        N, n = int(self.info.dataset_size), int(self.info.series_length)
        rows = np.empty((N, n), np.float32)
        words = np.empty((N, 16), np.uint8)
        orig = np.empty(N, np.uint32)
        _lib.call("ssb_index_download", self.handle, rows.ctypes.data_as(_lib.P),
                  words.ctypes.data_as(_lib.P), orig.ctypes.data_as(_lib.P))
        return rows, words, orig.astype(np.int64) + self.id_base

    def release_buffers(self) -> None:
        """build.py:161-171: nothing to release (no spill files or regions)."""


def build_index_array(data, settings, trace: BuildTrace | None = None, *, initial_segments: int = 1,
                      max_segments: int = 32, id_base: int = 0) -> SeriesIndex:
    """Build from an in-memory (N, n) block (numpy or torch; moved to the device)."""
    settings.validate()
    X = device_f32(data, settings.series_length)
    if X.shape[0] != settings.dataset_size:
        raise UsageError(f"data has {X.shape[0]} series, settings say {settings.dataset_size}")
    cfg = _lib.BuildCfg(int(settings.leaf_threshold), int(initial_segments), int(max_segments), int(id_base))
    raw = ctypes.c_void_p()
    _lib.call("ssb_build", ptr(X), X.shape[0], X.shape[1], ptr(device_breakpoints()), ctypes.byref(cfg),
              ctypes.byref(raw), stream_handle())
    idx = SeriesIndex(settings, _Handle(raw), trace)
    if trace is not None:
        for depth in range(idx.info.depth + 1):
            trace.note(0, "level", depth=depth)
        trace.note(0, "done", leaves=idx.info.num_leaves, levels=idx.info.levels,
                   build_ms=idx.info.build_ms)
    return idx


def ingest_file(path: str, n: int, first: int = 0, count: int | None = None, *,
                chunk_bytes: int = 64 << 20, threads: int = 0, stream=None):
    """Series [first, first + count) of a raw dataset file into HBM.

    The B200 form of the reference's chunked file reads feeding the build
    (build.py:414-451, DBuffer double buffering) and the scan (pscan.py:50-79):
    file -> pinned double buffer -> H2D copy, the read of chunk i overlapping the
    copy of chunk i-1 (csrc/ingest.cu).  Returns ``(tensor (count, n) float32 on
    the device, {"bytes", "seconds", "GBps"})``.  Missing file: DataFileError;
    size not a whole number of series or range past the end: UsageError.
    """
    t = require_cuda()
    total = series_count(path, n)  # DataFileError / UsageError before any allocation
    if first < 0 or first > total:
        raise UsageError(f"{path}: first series {first} outside [0, {total}]")
    if count is None:
        count = total - first
    if count < 0 or first + count > total:
        raise UsageError(f"{path}: requested series [{first}, {first + count}), file has {total}")
    X = t.empty((count, n), dtype=t.float32, device="cuda")
    st = (ctypes.c_double * 2)()
    _lib.call("ssb_ingest_file", path.encode(), int(first), int(count), int(n), ptr(X), int(chunk_bytes),
              int(threads), stream_handle(stream), st)
    secs = st[1]
    return X, {"bytes": int(st[0]), "seconds": secs, "GBps": (st[0] / secs / 1e9) if secs > 0 else None}


def build_index(dataset_path: str, settings, num_threads: int, buffer_bytes: int | None = None,
                dbsize: int | None = None, flush_threshold: int | None = None,
                scratch_dir: str | None = None, trace: BuildTrace | None = None, **kw) -> SeriesIndex:
    """Build the index from a raw dataset file (build.py:363-458 signature)."""
    settings.validate()
    n = settings.series_length
    data_size = series_count(dataset_path, n)
    if data_size != settings.dataset_size:
        raise UsageError(f"{dataset_path}: has {data_size} series, settings say {settings.dataset_size}")
    if num_threads < 2:
        raise UsageError("need at least 2 threads (coordinator + 1 worker)")
    num_workers = num_threads - 1
    if dbsize is None:
        dbsize = default_dbsize(data_size)
    if buffer_bytes is None:
        region_capacity = max(dbsize, math.ceil(data_size / num_workers) + dbsize)
    else:
        region_capacity = buffer_bytes // (4 * n * num_workers)
    if region_capacity < dbsize:
        raise UsageError(
            f"buffer too small: each of {num_workers} regions holds {region_capacity} series, "
            f"need at least one chunk of {dbsize}")
    # the file goes straight to HBM through the pinned double-buffer pipeline
    X, ingest = ingest_file(dataset_path, n, 0, data_size, threads=max(1, num_threads))
    if trace is not None:
        trace.note(0, "ingest", **ingest)
    return build_index_array(X, settings, trace, **kw)
