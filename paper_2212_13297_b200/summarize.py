"""Summarisation on the device: SAX words and EAPCA segment statistics.

Mirrors reference summarize.py (paths relative to
/root/reference/pkg/src/seriesearch): ``normal_breakpoints`` /
``symbol_bounds`` (:107-133) are host-side constants computed exactly as the
reference does (scipy ``norm.ppf``); ``paa_words`` replaces
``isax_from_paa(paa_batch(X, 16), bp)`` (:89-121) and
``segment_stats_matrix`` (:79-82) runs on the B200 (csrc/summarize.cu).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._device import device_f32, ptr, require_cuda, stream_handle
from .errors import UsageError

SUPPORTED_ALPHABETS = (2, 4, 8, 16, 32, 64, 128, 256)
WORD_SEGMENTS = 16

_bp_cache: dict = {}


def normal_breakpoints(alphabet_size: int = 256) -> np.ndarray:
    """Standard-normal quantiles at i/a, i = 1..a-1 (summarize.py:107-114).

    The 256-symbol table (the only alphabet the index uses, persist.py:84) is
    shipped pre-computed (_breakpoints.py, checked against scipy in the tests);
    other alphabets go through scipy like the reference."""
    if alphabet_size not in SUPPORTED_ALPHABETS:
        raise UsageError(
            f"alphabet size must be a power of two in [2, 256], got {alphabet_size}")
    if alphabet_size == 256:
        from ._breakpoints import BREAKPOINTS_256_HEX

        return np.array([float.fromhex(h) for h in BREAKPOINTS_256_HEX], dtype=np.float64)
    from scipy.stats import norm

    return norm.ppf(np.arange(1, alphabet_size) / alphabet_size)


def symbol_bounds(breakpoints: np.ndarray):
    """Per-symbol [lower, upper] with +-inf ends (summarize.py:124-133)."""
    a = breakpoints.size + 1
    lower = np.empty(a, dtype=np.float64)
    upper = np.empty(a, dtype=np.float64)
    lower[0] = -np.inf
    lower[1:] = breakpoints
    upper[: a - 1] = breakpoints
    upper[a - 1] = np.inf
    return lower, upper


def device_breakpoints():
    """The 255 breakpoints as a float64 CUDA tensor (cached per device)."""
    t = require_cuda()
    dev = t.cuda.current_device()
    if dev not in _bp_cache:
        _bp_cache[dev] = t.from_numpy(normal_breakpoints(256)).cuda()
    return _bp_cache[dev]


def paa_words(X, with_paa: bool = False):
    """SAX words (N, 16) uint8 [and PAA (N, 16) float32] of every row, on device."""
    t = require_cuda()
    x = device_f32(X)
    N, n = x.shape
    if n % WORD_SEGMENTS:
        raise UsageError(f"series length {n} is not divisible by {WORD_SEGMENTS} segments")
    words = t.empty((N, WORD_SEGMENTS), dtype=t.uint8, device=x.device)
    paa = t.empty((N, WORD_SEGMENTS), dtype=t.float32, device=x.device) if with_paa else None
    _lib.call("ssb_words", ptr(x), N, n, ptr(device_breakpoints()), ptr(words), ptr(paa),
              stream_handle())
    return (words, paa) if with_paa else words


def segment_stats_matrix(X, starts, ends):
    """Per-row mean/sd over segments [starts[j], ends[j]) -> two (N, m) float32
    CUDA tensors, bit-identical to summarize.py:79-82."""
    t = require_cuda()
    x = device_f32(X)
    N, n = x.shape
    s = np.ascontiguousarray(starts, dtype=np.int64)
    e = np.ascontiguousarray(ends, dtype=np.int64)
    if s.shape != e.shape or s.ndim != 1:
        raise UsageError("starts/ends must be equal-length 1-D arrays")
    m = s.size
    mean = t.empty((N, m), dtype=t.float32, device=x.device)
    sd = t.empty((N, m), dtype=t.float32, device=x.device)
    _lib.call("ssb_segment_stats", ptr(x), N, n, s.ctypes.data_as(_lib.P), e.ctypes.data_as(_lib.P),
              m, ptr(mean), ptr(sd), stream_handle())
    return mean, sd
