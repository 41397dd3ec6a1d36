"""Index settings, the queryable index, and the on-disk format.

Mirrors reference persist.py (/root/reference/pkg/src/seriesearch/persist.py):
``IndexSettings`` (:63-85), ``SeriesStore`` (:88-122), ``QueryableIndex``
(:125-138), ``write_index`` (:269-369) and ``load_index`` (:461-528), with the
same three files and byte layout (htree.bin header + postorder node records,
lrd.bin leaf-ordered rows, lsd.bin aligned words), so an index written here
loads in the reference and a reference-written index loads onto the GPU.
One extra file, ``ids.bin`` (uint64 original index per position), keeps the
original series indices; the reference ignores it and, when absent, positions
stand in for ids.
"""

from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DTYPE
from .errors import DataFileError, IntegrityError, UsageError
from .summarize import device_breakpoints, normal_breakpoints, symbol_bounds
from .tree import MEAN, Node, SplitPolicy

MAGIC = b"HTREEB01"
FORMAT_VERSION = 1
HTREE_NAME = "htree.bin"
LRD_NAME = "lrd.bin"
LSD_NAME = "lsd.bin"
IDS_NAME = "ids.bin"
_HEADER = struct.Struct("<8sIIQIIII")


@dataclass
class IndexSettings:
    series_length: int
    dataset_size: int
    leaf_threshold: int
    word_segments: int = 16
    alphabet_size: int = 256
    format_version: int = FORMAT_VERSION

    def validate(self) -> None:
        if self.series_length <= 0 or self.dataset_size <= 0:
            raise UsageError("series length and dataset size must be positive")
        if self.leaf_threshold <= 0:
            raise UsageError("leaf threshold must be positive")
        if self.word_segments <= 0 or self.series_length % self.word_segments != 0:
            raise UsageError(
                f"series length {self.series_length} is not divisible by "
                f"{self.word_segments} word segments")
        if self.alphabet_size != 256:
            raise UsageError("only the 256-symbol alphabet is supported on disk")
        if self.word_segments != 16:
            raise UsageError("the B200 path uses 16 word segments (persist.py:70 default)")


class SeriesStore:
    """Host view of the leaf-ordered rows with read accounting (persist.py:88-122).

    The device path never reads through it; queries report the rows they
    scanned through ``QueryStats`` instead.  ``data`` is copied from HBM on
    first use.
    """

    def __init__(self, fetch):
        self._fetch = fetch
        self._data = None
        self.series_read = 0
        self.read_seconds = 0.0

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            self._data = self._fetch()
        return self._data

    def read_slice(self, first: int, count: int) -> np.ndarray:
        self.series_read += count
        return np.asarray(self.data[first : first + count])

    def read_one(self, pos: int) -> np.ndarray:
        self.series_read += 1
        return np.asarray(self.data[pos])

    def reset_stats(self) -> None:
        self.series_read = 0
        self.read_seconds = 0.0


class QueryableIndex:
    """A written (or loaded) index, resident in HBM, ready for queries."""

    def __init__(self, settings: IndexSettings, series_index):
        self.settings = settings
        self.index = series_index          # build.SeriesIndex (owns the device handle)
        self.root: Node = series_index.root
        self.leaves = list(self.root.iter_leaves())
        self.total_leaves = len(self.leaves)
        self.total_series = settings.dataset_size
        self.breakpoints = normal_breakpoints(settings.alphabet_size)
        self.symbol_lower, self.symbol_upper = symbol_bounds(self.breakpoints)
        self._host = None
        self.store = SeriesStore(lambda: self._host_arrays()[0])

    def _host_arrays(self):
        if self._host is None:
            self._host = self.index.host_arrays()
        return self._host

    @property
    def words(self) -> np.ndarray:
        return self._host_arrays()[1]

    @property
    def ids(self) -> np.ndarray:
        """Original series index of every leaf-order position."""
        return self._host_arrays()[2]


# ---------------------------------------------------------------------------
# writing (persist.py:269-411)


def _node_record(node: Node) -> bytes:
    m = node.num_segments
    parts = [struct.pack("<BI", 1 if node.is_leaf else 0, m), node.endpoints.astype("<u4").tobytes()]
    syn = np.empty((m, 4), dtype=DTYPE)
    syn[:, 0], syn[:, 1], syn[:, 2], syn[:, 3] = node.mu_min, node.mu_max, node.sd_min, node.sd_max
    parts.append(syn.tobytes())
    parts.append(struct.pack("<Q", node.rho))
    if node.is_leaf:
        first, count = node.file_position
        parts.append(struct.pack("<QQ", first, count))
    else:
        p = node.policy
        parts.append(struct.pack("<IBBIIId", p.segment_index, 0 if p.attribute == MEAN else 1,
                                 1 if p.is_vsplit else 0, p.split_point if p.is_vsplit else 0,
                                 p.route_start, p.route_end, p.threshold))
    return b"".join(parts)


def _postorder(node: Node, out: list) -> None:
    if not node.is_leaf:
        _postorder(node.left, out)
        _postorder(node.right, out)
        node.rho = node.left.rho + node.right.rho
    out.append(_node_record(node))


def write_index(index, out_dir: str, num_threads: int = 1) -> QueryableIndex:
    """Materialise a built index to ``out_dir`` and return it query-ready."""
    settings = index.settings
    settings.validate()
    os.makedirs(out_dir, exist_ok=True)
    paths = [os.path.join(out_dir, nm) for nm in (LRD_NAME, LSD_NAME, HTREE_NAME, IDS_NAME)]
    rows, words, ids = index.host_arrays()
    try:
        records: list = []
        _postorder(index.root, records)
        with open(paths[0], "wb") as f:
            f.write(np.ascontiguousarray(rows, dtype=DTYPE).tobytes())
        with open(paths[1], "wb") as f:
            f.write(np.ascontiguousarray(words, dtype=np.uint8).tobytes())
        with open(paths[2], "wb") as f:
            f.write(_HEADER.pack(MAGIC, settings.format_version, settings.series_length,
                                 settings.dataset_size, settings.leaf_threshold, settings.word_segments,
                                 settings.alphabet_size, len(records)))
            for rec in records:
                f.write(rec)
        with open(paths[3], "wb") as f:
            f.write(ids.astype("<u8").tobytes())
    except OSError as exc:
        for p in paths:
            if os.path.exists(p):
                os.remove(p)
        raise DataFileError(f"index write failed: {exc}") from exc
    qi = QueryableIndex(settings, index)
    qi._host = (rows, words, ids)
    return qi


# ---------------------------------------------------------------------------
# loading (persist.py:414-528)


def _read_exact(f, size: int, path: str) -> bytes:
    data = f.read(size)
    if len(data) != size:
        raise IntegrityError(f"{path}: truncated (wanted {size} more bytes)")
    return data


def _read_tree(path: str):
    with open(path, "rb") as f:
        header = _read_exact(f, _HEADER.size, path)
        magic, version, n, dataset_size, tau, l, alphabet, num_nodes = _HEADER.unpack(header)
        if magic != MAGIC:
            raise IntegrityError(f"{path}: bad magic {magic!r}")
        if version != FORMAT_VERSION:
            raise IntegrityError(f"{path}: format version {version}, expected {FORMAT_VERSION}")
        settings = IndexSettings(series_length=n, dataset_size=dataset_size, leaf_threshold=tau,
                                 word_segments=l, alphabet_size=alphabet, format_version=version)
        try:
            settings.validate()
        except UsageError as exc:
            raise IntegrityError(f"{path}: bad settings: {exc}") from exc
        recs = []      # postorder records
        stack: list[int] = []
        children = {}
        for i in range(num_nodes):
            flags, m = struct.unpack("<BI", _read_exact(f, 5, path))
            ep = np.frombuffer(_read_exact(f, 4 * m, path), dtype="<u4").astype(np.int64)
            syn = np.frombuffer(_read_exact(f, 16 * m, path), dtype=DTYPE).reshape(m, 4)
            (rho,) = struct.unpack("<Q", _read_exact(f, 8, path))
            rec = {"m": m, "ep": ep, "syn": syn, "rho": rho, "leaf": bool(flags & 1)}
            if flags & 1:
                rec["first"], rec["count"] = struct.unpack("<QQ", _read_exact(f, 16, path))
            else:
                seg, attr, kind, sp, rs, re_, thr = struct.unpack("<IBBIIId", _read_exact(f, 26, path))
                rec.update(seg=seg, attr=attr, split=sp if kind == 1 else -1, rs=rs, re=re_, thr=thr)
                if len(stack) < 2:
                    raise IntegrityError(f"{path}: malformed postorder stream")
                r = stack.pop()
                lft = stack.pop()
                children[i] = (lft, r)
            recs.append(rec)
            stack.append(i)
        if f.read(1):
            raise IntegrityError(f"{path}: trailing bytes after tree")
    if len(stack) != 1:
        raise IntegrityError(f"{path}: postorder stream left {len(stack)} roots")
    return settings, recs, children, stack[0]


def load_index(index_dir: str) -> QueryableIndex:
    """Load a written index (ours or the reference's) onto the GPU."""
    from .build import SeriesIndex, _Handle

    htree, lrd, lsd = (os.path.join(index_dir, nm) for nm in (HTREE_NAME, LRD_NAME, LSD_NAME))
    for path in (htree, lrd, lsd):
        if not os.path.exists(path):
            raise IntegrityError(f"{path}: missing")
    settings, recs, children, root_i = _read_tree(htree)
    n, N, l = settings.series_length, settings.dataset_size, settings.word_segments
    if os.path.getsize(lrd) != N * n * 4:
        raise IntegrityError(f"{lrd}: size {os.path.getsize(lrd)}, expected {N * n * 4}")
    if os.path.getsize(lsd) != N * l:
        raise IntegrityError(f"{lsd}: size {os.path.getsize(lsd)}, expected {N * l}")
    rows = np.fromfile(lrd, dtype=DTYPE).reshape(N, n)
    words = np.fromfile(lsd, dtype=np.uint8).reshape(N, l)
    ids_path = os.path.join(index_dir, IDS_NAME)
    orig = None
    if os.path.exists(ids_path) and os.path.getsize(ids_path) == 8 * N:
        orig = np.fromfile(ids_path, dtype="<u8")
    # renumber: root first (preorder) -> node records for the C ABI
    order: list[int] = []
    stack = [root_i]
    while stack:
        i = stack.pop()
        order.append(i)
        if i in children:
            stack.append(children[i][1])
            stack.append(children[i][0])
    new_id = {old: k for k, old in enumerate(order)}
    NodeArr = _lib.NodeRec * len(order)
    arr = NodeArr()
    parent = {}
    for old, (lft, r) in children.items():
        parent[lft] = old
        parent[r] = old
    # member ranges: leaves carry (first, count); internal ranges from children
    first = {}
    count = {}
    depth = {root_i: 0}
    for old in order:
        if old in children:
            depth[children[old][0]] = depth[old] + 1
            depth[children[old][1]] = depth[old] + 1
    for old in reversed(order):
        rec = recs[old]
        if rec["leaf"]:
            first[old], count[old] = int(rec["first"]), int(rec["count"])
        else:
            lft, r = children[old]
            first[old] = min(first[lft], first[r])
            count[old] = count[lft] + count[r]
    for old in order:
        rec = recs[old]
        a = arr[new_id[old]]
        if rec["m"] > _lib.M_MAX:
            raise UsageError(f"node with {rec['m']} segments exceeds the device limit {_lib.M_MAX}")
        a.parent = new_id[parent[old]] if old in parent else -1
        a.left = new_id[children[old][0]] if old in children else -1
        a.right = new_id[children[old][1]] if old in children else -1
        a.first, a.count, a.m = first[old], count[old], rec["m"]
        for j in range(rec["m"]):
            a.endpoints[j] = int(rec["ep"][j])
            for q in range(4):
                a.envelope[j][q] = float(rec["syn"][j, q])
        a.is_leaf = 1 if rec["leaf"] else 0
        a.depth = depth[old]
        if not rec["leaf"]:
            a.segment, a.attribute, a.split_point = rec["seg"], rec["attr"], rec["split"]
            a.route_start, a.route_end, a.threshold = rec["rs"], rec["re"], rec["thr"]
        else:
            a.segment = -1
            a.split_point = -1
    raw = ctypes.c_void_p()
    orig32 = None if orig is None else np.ascontiguousarray(orig, dtype=np.uint32)
    _lib.call("ssb_index_load", rows.ctypes.data_as(_lib.P), words.ctypes.data_as(_lib.P),
              None if orig32 is None else orig32.ctypes.data_as(_lib.P), N, n,
              int(settings.leaf_threshold), 0, arr, len(order), ctypes.c_void_p(device_breakpoints().data_ptr()),
              ctypes.byref(raw), _stream())
    si = SeriesIndex(settings, _Handle(raw))
    qi = QueryableIndex(settings, si)
    qi._host = (rows, words, (np.arange(N, dtype=np.int64) if orig is None else orig.astype(np.int64)))
    return qi


def _stream():
    from ._device import stream_handle

    return stream_handle()
