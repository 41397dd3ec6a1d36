"""ctypes binding of libseriesearch_b200.so (include/seriesearch_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_2212_13297_b200/csrc``).  There is no CPU fallback: if the library or a
CUDA device is missing, every entry point raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import DataFileError, DeviceError, IntegrityError, UsageError

HERE = os.path.dirname(os.path.abspath(__file__))
# SSB_LIB_VARIANT=name loads libseriesearch_b200.<name>.so (A/B builds of the same sources)
LIB_PATH = os.path.join(HERE, "libseriesearch_b200.so" if not os.environ.get("SSB_LIB_VARIANT")
                        else "libseriesearch_b200.%s.so" % os.environ["SSB_LIB_VARIANT"])

_lib = None
_lock = threading.Lock()

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32

# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "ssb_version": [],
    "ssb_last_error": [],
    "ssb_launch_count": [],
    "ssb_device_ok": [],
    "ssb_prof_enable": [I32],
    "ssb_prof_reset": [],
    "ssb_prof_read": [I32, ctypes.c_char_p, I32, ctypes.POINTER(ctypes.c_double),
                      ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                      ctypes.POINTER(ctypes.c_double)],
    "ssb_words": [P, I64, I32, P, P, P, P],
    "ssb_segment_stats": [P, I64, I32, P, P, I32, P, P, P],
    "ssb_bruteforce_knn": [P, I64, I32, P, I32, I32, I64, P, P, P],
    "ssb_build": [P, I64, I32, P, P, P, P],
    "ssb_index_free": [P],
    "ssb_index_info": [P, P],
    "ssb_index_node": [P, I32, P],
    "ssb_index_arrays": [P, P, P, P, P],
    "ssb_query": [P, P, I32, I32, P, P, P, P, P, P],
    "ssb_query_multi": [P, I32, P, P, P, P, P, P, P, P],
    "ssb_tc_dot_debug": [P, I32, P, I64, I32, P, P],
    "ssb_index_download": [P, P, P, P],
    "ssb_index_load": [P, P, P, I64, I32, I64, I64, P, I32, P, P, P],
    "ssb_index_lb_eapca": [P, P, I32, P, P],
    "ssb_lb_sax": [P, P, I64, P, P, I32, P, P],
    "ssb_merge_topk": [P, I32, I32, I32, P, P, P],
    "ssb_pack_keys": [P, P, I64, P, P],
    "ssb_comm_unique_id": [P],
    "ssb_comm_init": [I32, I32, P, P],
    "ssb_comm_free": [P],
    "ssb_comm_merge_topk": [P, P, P, I32, I32, P, P, P],
    "ssb_index_set_comm": [P, P],
    "ssb_ingest_file": [ctypes.c_char_p, I64, I64, I32, P, I64, I32, P, P],
    "ssb_scan_file": [ctypes.c_char_p, I64, I64, I32, P, I32, I32, I64, I32, P, P, P, P],
    "ssb_generate": [I32, I64, I64, I32, ctypes.c_uint64, P, P],
}

M_MAX = 32


class BuildCfg(ctypes.Structure):
    _fields_ = [("leaf_threshold", ctypes.c_int64), ("initial_segments", ctypes.c_int32),
                ("max_segments", ctypes.c_int32), ("id_base", ctypes.c_int64)]


class QueryCfg(ctypes.Structure):
    _fields_ = [("eapca_th", ctypes.c_float), ("route", ctypes.c_int32), ("lmax", ctypes.c_int32)]


QUERY_STATS = 8  # SSB_QUERY_STATS columns per query


class IndexInfo(ctypes.Structure):
    _fields_ = [("dataset_size", ctypes.c_int64), ("leaf_threshold", ctypes.c_int64),
                ("id_base", ctypes.c_int64), ("series_length", ctypes.c_int32),
                ("num_nodes", ctypes.c_int32), ("num_leaves", ctypes.c_int32),
                ("levels", ctypes.c_int32), ("max_segments", ctypes.c_int32),
                ("depth", ctypes.c_int32), ("build_ms", ctypes.c_double),
                ("max_abs", ctypes.c_float), ("proj_dim", ctypes.c_int32), ("proj_energy", ctypes.c_double)]


class NodeRec(ctypes.Structure):
    _fields_ = [("parent", ctypes.c_int32), ("left", ctypes.c_int32), ("right", ctypes.c_int32),
                ("first", ctypes.c_uint32), ("count", ctypes.c_uint32), ("m", ctypes.c_int32),
                ("endpoints", ctypes.c_int32 * M_MAX), ("envelope", (ctypes.c_float * 4) * M_MAX),
                ("is_leaf", ctypes.c_int32), ("oversize", ctypes.c_int32), ("depth", ctypes.c_int32),
                ("segment", ctypes.c_int32), ("attribute", ctypes.c_int32),
                ("split_point", ctypes.c_int32), ("route_start", ctypes.c_int32),
                ("route_end", ctypes.c_int32), ("threshold", ctypes.c_double),
                ("gain", ctypes.c_double), ("inherited", ctypes.c_uint32), ("split_set", ctypes.c_uint32)]
_RESTYPES = {
    "ssb_version": ctypes.c_int32,
    "ssb_last_error": ctypes.c_char_p,
    "ssb_launch_count": ctypes.c_int64,
    "ssb_device_ok": ctypes.c_int32,
    "ssb_prof_enable": None,
    "ssb_prof_reset": None,
}


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def load():
    """Load (once) and return the CDLL; raises DeviceError if absent."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, args in _SIGS.items():
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = lib
    return _lib


_ERRORS = {1: UsageError, 2: DataFileError, 3: IntegrityError, 4: DeviceError, 5: DeviceError}


def call(name: str, *args) -> None:
    """Invoke an ``int``-returning entry point; map its code to an exception."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.ssb_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, DeviceError)(f"{name}: {msg}")


def launch_count() -> int:
    return int(load().ssb_launch_count())


def prof_enable(on: bool = True) -> None:
    load().ssb_prof_enable(1 if on else 0)


def prof_reset() -> None:
    load().ssb_prof_reset()


def prof_read() -> dict:
    """{kernel: (ms_total, launches, algorithmic_bytes_total, algorithmic_flops_total)}."""
    lib = load()
    out = {}
    i = 0
    buf = ctypes.create_string_buffer(64)
    while True:
        ms, n, b, f = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
        if lib.ssb_prof_read(i, buf, 64, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b),
                             ctypes.byref(f)) != 0:
            break
        out[buf.value.decode()] = (ms.value, n.value, b.value, f.value)
        i += 1
    return out
