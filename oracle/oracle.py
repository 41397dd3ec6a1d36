"""CPU oracle for the exact k-NN data-series search path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this module, and only as
the checker (or the timed CPU baseline).  The product package
``paper_2212_13297_b200`` never imports it.

It wraps ``libssb_oracle.so`` (``ssb_oracle.c``, a plain-C restatement of the
reference's numpy arithmetic) and adds a few numpy restatements for the cases
where numpy itself is the clearest statement.  Every function cites the
reference file:line it follows (paths relative to
``/root/reference/pkg/src/seriesearch``).

Pinning: ``tests/test_oracle.py`` checks every function here against golden
vectors that ``tests/golden/make_golden.py`` produced by running the reference
package itself (see that script).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libssb_oracle.so")
_lib = None


def build() -> str:
    """Compile the C oracle in place (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


class Policy(ctypes.Structure):
    _fields_ = [
        ("segment_index", ctypes.c_int32),
        ("attribute", ctypes.c_int32),
        ("split_point", ctypes.c_int32),
        ("route_start", ctypes.c_int32),
        ("route_end", ctypes.c_int32),
        ("n_left", ctypes.c_int32),
        ("threshold", ctypes.c_double),
        ("gain", ctypes.c_double),
    ]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        L.ssbo_ed2_rows.argtypes = [P, i64, i32, P, P]
        L.ssbo_knn_scan.argtypes = [P, i64, i32, P, i32, i32, P, P, i32]
        L.ssbo_knn_scan.restype = ctypes.c_int
        L.ssbo_segment_stats.argtypes = [P, i64, i32, P, P, i32, P, P]
        L.ssbo_paa.argtypes = [P, i64, i32, i32, P]
        L.ssbo_sax.argtypes = [P, i64, P, i32, P]
        L.ssbo_lb_sax.argtypes = [P, i32, P, i64, P, P, i32, P]
        L.ssbo_lb_eapca.argtypes = [P, P, P, i32, P, P, P, P]
        L.ssbo_lb_eapca.restype = ctypes.c_double
        L.ssbo_lb_eapca_query.argtypes = [P, i32, P, i32, P, P, P, P]
        L.ssbo_lb_eapca_query.restype = ctypes.c_double
        L.ssbo_best_split.argtypes = [P, i64, i32, P, i32, ctypes.c_float, ctypes.c_float,
                                      i32, ctypes.POINTER(Policy)]
        L.ssbo_best_split.restype = ctypes.c_int
        L.ssbo_policy_size.restype = ctypes.c_int32
        assert L.ssbo_policy_size() == ctypes.sizeof(Policy)
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# ---------------------------------------------------------------------------
# core.py:50-57 ed2_batch


def ed2_rows(X, q) -> np.ndarray:
    X = _f32(np.atleast_2d(X))
    q = _f32(q)
    out = np.empty(X.shape[0], np.float32)
    lib().ssbo_ed2_rows(_p(X), X.shape[0], X.shape[1], _p(q), _p(out))
    return out


def ed2_numpy(X, q) -> np.ndarray:
    """core.py:50-57 verbatim numpy form (the reference's own expression)."""
    d = _f32(X) - _f32(q)
    return (d * d).sum(axis=-1)


# ---------------------------------------------------------------------------
# pscan.py:23-30 brute_force_knn (ties -> lowest row index)


def knn_scan(X, Q, k: int, threads: int = 1):
    """Exact k-NN of every query row of Q over X.

    Returns (d2 (B,k) float32, ids (B,k) int64); missing entries are (inf, -1).
    """
    X = _f32(np.atleast_2d(X))
    Q = _f32(np.atleast_2d(Q))
    B = Q.shape[0]
    d2 = np.empty((B, k), np.float32)
    ids = np.empty((B, k), np.int64)
    rc = lib().ssbo_knn_scan(_p(X), X.shape[0], X.shape[1], _p(Q), B, k, _p(d2), _p(ids),
                             max(1, int(threads)))
    if rc != 0:
        raise ValueError("ssbo_knn_scan rejected its arguments")
    return d2, ids


def knn_numpy(X, q, k: int):
    """pscan.py:23-30: ed2_batch + stable argsort, first k (small cases)."""
    d = ed2_numpy(X, q)
    order = np.argsort(d, kind="stable")[:k]
    return d[order], order.astype(np.int64)


# ---------------------------------------------------------------------------
# summarize.py:34-82 EAPCA statistics


def segment_stats(X, starts, ends):
    X = _f32(np.atleast_2d(X))
    starts = np.ascontiguousarray(starts, np.int64)
    ends = np.ascontiguousarray(ends, np.int64)
    m = starts.size
    mean = np.empty((X.shape[0], m), np.float32)
    sd = np.empty((X.shape[0], m), np.float32)
    lib().ssbo_segment_stats(_p(X), X.shape[0], X.shape[1], _p(starts), _p(ends), m,
                             _p(mean), _p(sd))
    return mean, sd


# ---------------------------------------------------------------------------
# summarize.py:89-133 PAA, breakpoints, SAX words, symbol bounds


def paa(X, l: int = 16):
    X = _f32(np.atleast_2d(X))
    out = np.empty((X.shape[0], l), np.float32)
    lib().ssbo_paa(_p(X), X.shape[0], X.shape[1], l, _p(out))
    return out


def normal_breakpoints(alphabet: int = 256) -> np.ndarray:
    """summarize.py:107-114: scipy.stats.norm.ppf(i/alphabet), i = 1..a-1."""
    from scipy.stats import norm

    return norm.ppf(np.arange(1, alphabet) / alphabet)


def symbol_bounds(bp: np.ndarray):
    """summarize.py:124-133: per-symbol [lower, upper] with +-inf ends."""
    a = bp.size + 1
    lower = np.empty(a)
    upper = np.empty(a)
    lower[0] = -np.inf
    lower[1:] = bp
    upper[: a - 1] = bp
    upper[a - 1] = np.inf
    return lower, upper


def sax(paa_values, bp) -> np.ndarray:
    p = _f32(paa_values)
    bp = np.ascontiguousarray(bp, np.float64)
    out = np.empty(p.shape, np.uint8)
    lib().ssbo_sax(_p(p), p.size, _p(bp), bp.size, _p(out))
    return out


def words(X, bp, l: int = 16):
    return sax(paa(X, l), bp)


# ---------------------------------------------------------------------------
# summarize.py:136-153 LB_SAX ; 170-206 LB_EAPCA


def lb_sax(qpaa, W, lower, upper, n: int) -> np.ndarray:
    qpaa = _f32(qpaa)
    W = np.ascontiguousarray(W, np.uint8)
    lower = np.ascontiguousarray(lower, np.float64)
    upper = np.ascontiguousarray(upper, np.float64)
    out = np.empty(W.shape[0], np.float64)
    lib().ssbo_lb_sax(_p(qpaa), qpaa.size, _p(W), W.shape[0], _p(lower), _p(upper), n, _p(out))
    return out


def lb_eapca(qmeans, qsds, widths, mu_min, mu_max, sd_min, sd_max) -> float:
    a = [_f32(qmeans), _f32(qsds)]
    w = np.ascontiguousarray(widths, np.float64)
    e = [_f32(v) for v in (mu_min, mu_max, sd_min, sd_max)]
    return float(lib().ssbo_lb_eapca(_p(a[0]), _p(a[1]), _p(w), w.size, *[_p(v) for v in e]))


def lb_eapca_query(q, endpoints, mu_min, mu_max, sd_min, sd_max) -> float:
    q = _f32(q)
    ep = np.ascontiguousarray(endpoints, np.int64)
    e = [_f32(v) for v in (mu_min, mu_max, sd_min, sd_max)]
    return float(lib().ssbo_lb_eapca_query(_p(q), q.size, _p(ep), ep.size, *[_p(v) for v in e]))


# ---------------------------------------------------------------------------
# tree.py:211-336 get_best_split_policy


def best_split(members, endpoints, mu_min0=np.inf, mu_max0=-np.inf, allow_vsplit=True) -> dict:
    M = _f32(np.atleast_2d(members))
    ep = np.ascontiguousarray(endpoints, np.int64)
    pol = Policy()
    rc = lib().ssbo_best_split(_p(M), M.shape[0], M.shape[1], _p(ep), ep.size,
                               ctypes.c_float(mu_min0), ctypes.c_float(mu_max0),
                               1 if allow_vsplit else 0, ctypes.byref(pol))
    if rc != 0:
        raise ValueError("ssbo_best_split rejected its arguments")
    return {
        "segment_index": pol.segment_index,
        "attribute": "mean" if pol.attribute == 0 else "sd",
        "split_point": None if pol.split_point < 0 else pol.split_point,
        "route_start": pol.route_start,
        "route_end": pol.route_end,
        "threshold": pol.threshold,
        "gain": pol.gain,
        "n_left": pol.n_left,
    }


# ---------------------------------------------------------------------------
# device generator stream (csrc/generate.cu).  The reference's
# generator is numpy's Philox(SeedSequence(seed, spawn_key=(i,))) (generate.py:
# 27-81); the device generator keeps its recipe (walk = cumsum of N(0,1) in
# float64 -> float32 -> z_normalize, core.py:33-47; unit rows = N(0,1) / L2
# norm) on a documented NEW stream, restated here in numpy.  Philox4x32-10 is
# pinned by the Random123 known-answer vectors (tests/test_oracle.py).

_PH_M = (np.uint64(0xD2511F53), np.uint64(0xCD9E8D57))
_PH_W = (0x9E3779B9, 0xBB67AE85)


def philox4x32_10(ctr, key):
    """Philox4x32-10 (Salmon et al. SC'11) on arrays: ctr (..., 4) u32, key (2,) u32 -> (..., 4) u32."""
    c = np.asarray(ctr, np.uint64).copy()
    k0, k1 = int(key[0]), int(key[1])
    m32 = np.uint64(0xFFFFFFFF)
    for r in range(10):
        if r:
            k0 = (k0 + _PH_W[0]) & 0xFFFFFFFF
            k1 = (k1 + _PH_W[1]) & 0xFFFFFFFF
        p0 = _PH_M[0] * c[..., 0]
        p1 = _PH_M[1] * c[..., 2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c = np.stack([hi1 ^ c[..., 1] ^ np.uint64(k0), lo1, hi0 ^ c[..., 3] ^ np.uint64(k1), lo0], axis=-1)
    return c.astype(np.uint32)


def gen_normals(start: int, count: int, n: int, seed: int, tag: int) -> np.ndarray:
    """(count, n) float64 normals of the device stream (generate.cu gen_normal)."""
    i = np.arange(start, start + count, dtype=np.uint64)[:, None]
    b = np.arange((n + 1) // 2, dtype=np.uint64)[None, :]
    ctr = np.stack(np.broadcast_arrays(b, i & np.uint64(0xFFFFFFFF), i >> np.uint64(32),
                                       np.full_like(b, tag)), axis=-1)
    x = philox4x32_10(ctr, (seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)).astype(np.float64)
    u1 = (np.floor(x[..., 0] / 32) * 67108864.0 + np.floor(x[..., 1] / 64) + 0.5) / 9007199254740992.0
    u2 = (np.floor(x[..., 2] / 32) * 67108864.0 + np.floor(x[..., 3] / 64) + 0.5) / 9007199254740992.0
    r = np.sqrt(-2.0 * np.log(u1))
    z = np.empty((count, 2 * b.shape[1]))
    z[:, 0::2] = r * np.cos(2 * np.pi * u2)
    z[:, 1::2] = r * np.sin(2 * np.pi * u2)
    return z[:, :n]


def gen_random_walks(start: int, count: int, n: int, seed: int) -> np.ndarray:
    """Device stream kind 0: z_normalize(f32(cumsum(normals))) per series (core.py:33-47)."""
    w = np.cumsum(gen_normals(start, count, n, seed, 0), axis=1).astype(np.float32).astype(np.float64)
    mu = w.mean(axis=1, keepdims=True)
    sd = w.std(axis=1, keepdims=True)
    out = ((w - mu) / np.where(sd < 1e-8, 1.0, sd)).astype(np.float32)
    out[(sd < 1e-8)[:, 0]] = 0
    return out


def gen_unit_gaussian(start: int, count: int, n: int, seed: int) -> np.ndarray:
    """Device stream kind 1: normals / float64 L2 norm, float32."""
    z = gen_normals(start, count, n, seed, 1)
    return (z / np.linalg.norm(z, axis=1, keepdims=True)).astype(np.float32)
