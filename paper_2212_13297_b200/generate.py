"""Seeded synthetic series (harness data producer, not a device kernel).

Restates reference generate.py (/root/reference/pkg/src/seriesearch/
generate.py:27-81) so benchmarks and tests use the configs' own inputs:
series ``i`` of a seed comes from ``Philox(SeedSequence(seed, spawn_key=(i,)))``
-> cumsum of N(0,1) in float64 -> float32 -> z-normalised (core.py:33-47),
so any prefix is byte-identical to the reference generator.  Large datasets
are produced in parallel worker processes by row range (the stream is
prefix-stable), which is the only change.

``noise_queries`` follows generate_noise_workload (:58-81) but takes the
noise standard deviation directly (BASELINE.json configs quote sigma in
{0.01, 0.1, 1.0}; the reference function only admits variances in
[0.01, 0.1]).  ``unit_gaussian_block`` is the config-3 stand-in for 96-d
embeddings (no reference generator exists).
"""

from __future__ import annotations

import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

from .core import DTYPE, z_normalize


def _series_rng(seed: int, i: int) -> np.random.Generator:
    ss = np.random.SeedSequence(entropy=seed, spawn_key=(i,))
    return np.random.Generator(np.random.Philox(ss))


def random_walk_block(start: int, count: int, n: int, seed: int) -> np.ndarray:
    """Series [start, start+count) of the seeded random-walk stream."""
    out = np.empty((count, n), dtype=DTYPE)
    for j in range(count):
        rng = _series_rng(seed, start + j)
        walk = np.cumsum(rng.standard_normal(n))
        out[j] = z_normalize(walk.astype(DTYPE))
    return out


def _rw_chunk(args):
    start, count, n, seed = args
    return start, random_walk_block(start, count, n, seed)


def random_walks(count: int, n: int, seed: int, workers: int | None = None,
                 chunk: int = 8192, start: int = 0) -> np.ndarray:
    """Series [start, start+count) of the stream, generated in parallel
    (prefix-stable: any row range equals the same rows of the full dataset)."""
    out = np.empty((count, n), dtype=DTYPE)
    jobs = [(start + s, min(chunk, count - s), n, seed) for s in range(0, count, chunk)]
    workers = workers or min(len(jobs), os.cpu_count() or 1)
    if workers <= 1 or len(jobs) == 1:
        for job in jobs:
            s, blk = _rw_chunk(job)
            out[s - start : s - start + len(blk)] = blk
        return out
    with ProcessPoolExecutor(max_workers=workers) as ex:
        for s, blk in ex.map(_rw_chunk, jobs):
            out[s - start : s - start + len(blk)] = blk
    return out


def noise_queries_stream(total: int, n: int, count: int, sigma: float, seed: int,
                         data_seed: int = 0) -> np.ndarray:
    """``noise_queries`` over the random-walk dataset (total, n, data_seed)
    without materialising it: each query's source row is regenerated from the
    prefix-stable stream (identical to noise_queries(X, ...))."""
    queries = np.empty((count, n), dtype=DTYPE)
    for j in range(count):
        rng = _series_rng(seed, j)
        src = int(rng.integers(total))
        row = random_walk_block(src, 1, n, data_seed)[0]
        noisy = row.astype(np.float64) + rng.normal(0.0, sigma, n)
        queries[j] = z_normalize(noisy.astype(DTYPE))
    return queries


def noise_queries(data: np.ndarray, count: int, sigma: float, seed: int) -> np.ndarray:
    """Query j: rng=_series_rng(seed, j); src=rng.integers(N);
    z_normalize(f32(data[src] + rng.normal(0, sigma, n))) (generate.py:58-81)."""
    total, n = data.shape
    queries = np.empty((count, n), dtype=DTYPE)
    for j in range(count):
        rng = _series_rng(seed, j)
        src = int(rng.integers(total))
        noisy = data[src].astype(np.float64) + rng.normal(0.0, sigma, n)
        queries[j] = z_normalize(noisy.astype(DTYPE))
    return queries


def unit_gaussian_rows(lo: int, hi: int, n: int, seed: int, chunk: int = 65536,
                       workers: int | None = None) -> np.ndarray:
    """Rows [lo, hi) of unit_gaussian(total, n, seed) (chunk-aligned generation)."""
    c0, c1 = lo // chunk, (hi + chunk - 1) // chunk
    jobs = [(c, chunk, n, seed) for c in range(c0, c1)]
    out = np.empty(((c1 - c0) * chunk, n), dtype=DTYPE)
    workers = workers or min(len(jobs), os.cpu_count() or 1)
    if workers <= 1 or len(jobs) <= 1:
        for job in jobs:
            c, blk = _ug_chunk(job)
            out[(c - c0) * chunk : (c - c0) * chunk + len(blk)] = blk
    else:
        with ProcessPoolExecutor(max_workers=workers) as ex:
            for c, blk in ex.map(_ug_chunk, jobs):
                out[(c - c0) * chunk : (c - c0) * chunk + len(blk)] = blk
    return out[lo - c0 * chunk : hi - c0 * chunk]


def _ug_chunk(args):
    c, rows, n, seed = args
    rng = np.random.Generator(np.random.Philox(np.random.SeedSequence(seed, spawn_key=(c,))))
    v = rng.standard_normal((rows, n))
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return c, v.astype(DTYPE)


def unit_gaussian(count: int, n: int, seed: int, chunk: int = 65536,
                  workers: int | None = None) -> np.ndarray:
    """i.i.d. N(0,1) rows L2-normalised in float64, then float32; chunk c of
    65,536 rows draws from Philox(SeedSequence(seed, spawn_key=(c,)))."""
    out = np.empty((count, n), dtype=DTYPE)
    jobs = [(c, min(chunk, count - c * chunk), n, seed)
            for c in range((count + chunk - 1) // chunk)]
    workers = workers or min(len(jobs), os.cpu_count() or 1)
    if workers <= 1 or len(jobs) == 1:
        for job in jobs:
            c, blk = _ug_chunk(job)
            out[c * chunk : c * chunk + len(blk)] = blk
        return out
    with ProcessPoolExecutor(max_workers=workers) as ex:
        for c, blk in ex.map(_ug_chunk, jobs):
            out[c * chunk : c * chunk + len(blk)] = blk
    return out


def _device_series(kind: int, count: int, n: int, seed: int, start: int, stream):
    import ctypes

    from . import _lib
    from ._device import ptr, require_cuda, stream_handle

    t = require_cuda()
    out = t.empty((count, n), dtype=t.float32, device="cuda")
    _lib.call("ssb_generate", int(kind), int(start), int(count), int(n), ctypes.c_uint64(seed & (2**64 - 1)),
              ptr(out), stream_handle(stream))
    return out


def random_walks_device(count: int, n: int, seed: int, start: int = 0, stream=None):
    """Series [start, start+count) of the DEVICE random-walk stream, in HBM.

    Same recipe as ``random_walks`` (float64 cumsum of N(0,1) -> float32 ->
    z-normalised, generate.py:42-55 / core.py:33-47) on a documented new
    stream: Philox4x32-10 + Box-Muller (csrc/generate.cu), not numpy's bits.
    Prefix-stable, so each rank of a sharded build generates only its rows.
    """
    return _device_series(0, count, n, seed, start, stream)


def unit_gaussian_device(count: int, n: int, seed: int, start: int = 0, stream=None):
    """Rows [start, start+count) of the DEVICE unit-Gaussian stream (N(0,1) / L2 norm)."""
    return _device_series(1, count, n, seed, start, stream)
