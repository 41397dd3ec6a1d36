"""Host-side summarisation constants (CPU)."""

import numpy as np
import pytest

from conftest import golden


def test_breakpoint_table_equals_scipy_and_reference():
    from scipy.stats import norm

    from paper_2212_13297_b200.summarize import normal_breakpoints, symbol_bounds

    bp = normal_breakpoints(256)
    assert np.array_equal(bp, norm.ppf(np.arange(1, 256) / 256))
    g = golden("words")
    assert np.array_equal(bp, g["bp"])
    lo, hi = symbol_bounds(bp)
    assert np.array_equal(lo, g["lower"]) and np.array_equal(hi, g["upper"])


@pytest.mark.parametrize("a", [2, 4, 16, 256])
def test_other_alphabets(a):
    from paper_2212_13297_b200.summarize import normal_breakpoints

    bp = normal_breakpoints(a)
    assert len(bp) == a - 1 and np.all(np.diff(bp) > 0)


def test_bad_alphabet():
    from paper_2212_13297_b200 import UsageError
    from paper_2212_13297_b200.summarize import normal_breakpoints

    with pytest.raises(UsageError):
        normal_breakpoints(3)
