"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import golden, random_walks


def test_ed2_bitwise(oracle):
    g = golden("ed2")
    for n in (16, 64, 96, 256, 320):
        got = oracle.ed2_rows(g[f"X{n}"], g[f"q{n}"])
        assert np.array_equal(got.view(np.uint32), g[f"d2_{n}"].view(np.uint32)), n


def test_ed2_numpy_restatement_matches_c(oracle):
    X = random_walks(500, 256, 1)
    q = random_walks(1, 256, 2)[0]
    assert np.array_equal(oracle.ed2_rows(X, q), oracle.ed2_numpy(X, q))


@pytest.mark.parametrize("k", [1, 10, 100])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_knn_scan_matches_reference_brute_force(oracle, k, threads):
    g = golden("knn")
    d2, ids = oracle.knn_scan(g["X"], g["Q"], k, threads=threads)
    assert np.array_equal(d2, g[f"d2_k{k}"])
    assert np.array_equal(ids, g[f"id_k{k}"])


def test_knn_ties_go_to_lowest_index(oracle):
    g = golden("knn")
    d2, ids = oracle.knn_scan(g["X"], g["Q"], 3)
    # query 6 is row 10, duplicated at rows 2500 and 2999
    assert list(ids[6]) == [10, 2500, 2999] and d2[6][0] == 0.0
    assert list(ids[7][:2]) == [1100, 1200]


def test_knn_pads_when_k_exceeds_rows(oracle):
    X = random_walks(5, 32, 3)
    d2, ids = oracle.knn_scan(X, X[:1], 8)
    assert list(ids[0][5:]) == [-1, -1, -1] and np.isinf(d2[0][5:]).all()


def test_segment_stats_bitwise(oracle):
    g = golden("stats")
    for name in ("root", "three", "fine", "width1"):
        mean, sd = oracle.segment_stats(g["X"], g[f"starts_{name}"], g[f"ends_{name}"])
        assert np.array_equal(mean, g[f"mean_{name}"]), name
        assert np.array_equal(sd, g[f"sd_{name}"]), name


def test_breakpoints_and_words_bitwise(oracle):
    g = golden("words")
    bp = oracle.normal_breakpoints(256)
    assert np.array_equal(bp, g["bp"])
    lo, hi = oracle.symbol_bounds(bp)
    assert np.array_equal(lo, g["lower"]) and np.array_equal(hi, g["upper"])
    for n in (96, 256):
        p = oracle.paa(g[f"X{n}"], 16)
        assert np.array_equal(p, g[f"paa{n}"]), n
        assert np.array_equal(oracle.sax(p, bp), g[f"words{n}"]), n


def test_lb_sax_bitwise(oracle):
    g = golden("lbsax")
    lo, hi = oracle.symbol_bounds(oracle.normal_breakpoints(256))
    for i, qp in enumerate(g["qpaa"]):
        got = oracle.lb_sax(qp, g["W"], lo, hi, int(g["n"]))
        assert np.array_equal(got, g["lb"][i])


def test_lb_eapca_bitwise(oracle):
    g = golden("lbeapca")
    for i in range(int(g["count"])):
        got = oracle.lb_eapca_query(g[f"q{i}"], g[f"ep{i}"], g[f"mu_min{i}"], g[f"mu_max{i}"],
                                    g[f"sd_min{i}"], g[f"sd_max{i}"])
        assert got == float(g[f"lb{i}"]), i


def test_lb_eapca_worked_example(oracle):
    # reference tests/test_summarize.py:172-179 -> 16.16
    got = oracle.lb_eapca([0.0], [1.0], [4.0], [2.0], [3.0], [0.5], [0.8])
    assert got == pytest.approx(16.16, abs=1e-6)


def test_best_split_matches_reference(oracle):
    g = golden("split")
    for c in range(int(g["count"])):
        pol = oracle.best_split(g[f"members{c}"], g[f"ep{c}"], float(g[f"mu_min0_{c}"]),
                                float(g[f"mu_max0_{c}"]))
        seg, attr, sp, rs, re_ = (int(v) for v in g[f"pol{c}"])
        assert pol["segment_index"] == seg, c
        assert pol["attribute"] == ("mean" if attr == 0 else "sd"), c
        assert (pol["split_point"] if pol["split_point"] is not None else -1) == sp, c
        assert (pol["route_start"], pol["route_end"]) == (rs, re_), c
        assert pol["threshold"] == float(g[f"thr{c}"]), c
        assert pol["gain"] == float(g[f"gain{c}"]), c
        assert pol["n_left"] == int(g[f"nleft{c}"]), c


def test_reference_engine_equals_oracle_scan(oracle):
    """The reference's own index engine (build/write/exact_knn) answered these
    queries; its distances must equal the oracle's full scan."""
    g = golden("engine")
    for k in (1, 10):
        d2, _ = oracle.knn_scan(g["data"], g["queries"], k)
        assert np.array_equal(d2, g[f"d2_k{k}"]), k


def test_philox_known_answers(oracle):
    """Random123 kat_vectors for philox4x32-10 (the device generator's stream)."""
    import numpy as np

    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        got = oracle.philox4x32_10(np.array(ctr, np.uint32), key)
        assert tuple(int(v) for v in got) == want
