"""CPU-side checks of the C-ABI boundary: the library loads and exports every
symbol include/seriesearch_b200.h declares (no compute without a GPU)."""

import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "seriesearch_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ssb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for required in ("ssb_bruteforce_knn", "ssb_words", "ssb_segment_stats", "ssb_last_error"):
        assert required in syms


def test_library_exports_every_declared_symbol():
    from paper_2212_13297_b200 import _lib

    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
        # ctypes resolves through dlsym; a missing export raises AttributeError
        assert isinstance(getattr(lib, name), ctypes._CFuncPtr)


def test_bindings_cover_header():
    from paper_2212_13297_b200 import _lib

    assert set(declared_symbols()) == set(_lib.exported_symbols())


def test_library_is_sm100a_only():
    import subprocess

    from paper_2212_13297_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:  # cuobjdump missing: nothing to check
        return
    assert "sm_100a" in out.stdout
    assert "sm_90" not in out.stdout


def test_no_device_means_loud_failure():
    import numpy as np
    import pytest
    import torch

    from paper_2212_13297_b200 import DeviceError, brute_force_knn

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(DeviceError):
        brute_force_knn(np.zeros((4, 16), np.float32), np.zeros(16, np.float32), 1)
