"""Host-side checks of the ingest pipeline's file validation (csrc/ingest.cu):
the C entry point rejects a missing file (io, DataFileError) and a file that is
not a whole number of series or a range past its end (usage, UsageError) before
touching the device, like core.py series_count / read_series_file."""

import ctypes

import numpy as np
import pytest


def _call(path, first, count, n):
    from paper_2212_13297_b200 import _lib

    lib = _lib.load()
    rc = lib.ssb_ingest_file(str(path).encode(), first, count, n, None, 0, 1, None, None)
    return rc, lib.ssb_last_error().decode()


def test_missing_file_is_io_error(tmp_path):
    rc, msg = _call(tmp_path / "nope.bin", 0, -1, 16)
    assert rc == 2 and "nope.bin" in msg


def test_ragged_file_is_usage_error(tmp_path):
    p = tmp_path / "ragged.bin"
    np.zeros(16 * 3 + 5, np.float32).tofile(p)
    rc, msg = _call(p, 0, -1, 16)
    assert rc == 1 and "not a multiple" in msg


@pytest.mark.parametrize("first,count", [(0, 4), (3, 2), (5, -1)])
def test_range_past_end_is_usage_error(tmp_path, first, count):
    p = tmp_path / "three.bin"
    np.zeros((3, 16), np.float32).tofile(p)
    rc, msg = _call(p, first, count, 16)
    assert rc == 1 and "file has 3" in msg


def test_empty_range_needs_no_device(tmp_path):
    p = tmp_path / "three.bin"
    np.zeros((3, 16), np.float32).tofile(p)
    assert _call(p, 3, 0, 16)[0] == 0
    assert _call(p, 1, 0, 16)[0] == 0


def test_python_wrapper_maps_errors(tmp_path):
    import paper_2212_13297_b200 as ssb
    from paper_2212_13297_b200 import DataFileError, DeviceError, UsageError

    with pytest.raises((DataFileError, DeviceError)):
        ssb.ingest_file(str(tmp_path / "missing.bin"), 16)
    p = tmp_path / "ragged.bin"
    np.zeros(17, np.float32).tofile(p)
    with pytest.raises((UsageError, DeviceError)):
        ssb.ingest_file(str(p), 16)
