"""The harness generator reproduces the reference generator byte for byte
(golden vectors from the reference's generate.py)."""

import numpy as np

from conftest import golden


def test_random_walks_match_reference():
    from paper_2212_13297_b200 import generate as G

    g = golden("generate")
    assert np.array_equal(G.random_walk_block(0, 6, 256, 0), g["walk256_s0"])
    assert np.array_equal(G.random_walk_block(1000, 3, 256, 0), g["walk256_s0_at1000"])
    assert np.array_equal(G.random_walk_block(5, 4, 96, 3), g["walk96_s3"])


def test_parallel_generation_is_prefix_stable():
    from paper_2212_13297_b200 import generate as G

    a = G.random_walks(50, 64, 0, workers=2, chunk=16)
    assert np.array_equal(a, G.random_walk_block(0, 50, 64, 0))
    g = golden("generate")
    assert np.array_equal(a, g["noise_base"])


def test_noise_queries_match_reference_recipe():
    from paper_2212_13297_b200 import generate as G

    g = golden("generate")
    for sigma in (0.01, 0.1, 1.0):
        q = G.noise_queries(g["noise_base"], 5, sigma, 1)
        assert np.array_equal(q, g[f"noise_q_{sigma}"]), sigma


def test_unit_gaussian_rows_are_unit():
    from paper_2212_13297_b200 import generate as G

    x = G.unit_gaussian(1000, 96, 2, chunk=300, workers=1)
    assert np.allclose(np.linalg.norm(x.astype(np.float64), axis=1), 1.0, atol=1e-6)
    assert np.array_equal(x, G.unit_gaussian(1000, 96, 2, chunk=300, workers=2))


def test_sharded_generation_matches_full():
    from paper_2212_13297_b200 import generate as G

    full = G.random_walks(40, 32, 0, workers=1)
    assert np.array_equal(G.random_walks(15, 32, 0, workers=2, chunk=4, start=20), full[20:35])
    assert np.array_equal(G.random_walks(15, 32, 0, workers=1, chunk=4, start=20), full[20:35])
    q1 = G.noise_queries(full, 6, 0.1, 1)
    q2 = G.noise_queries_stream(40, 32, 6, 0.1, 1, data_seed=0)
    assert np.array_equal(q1, q2)
    u = G.unit_gaussian(3000, 16, 2, chunk=500, workers=1)
    assert np.array_equal(G.unit_gaussian_rows(1234, 2777, 16, 2, chunk=500, workers=2), u[1234:2777])
