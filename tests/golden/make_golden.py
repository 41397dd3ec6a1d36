"""Generate the golden vectors that pin the CPU oracle (and the CUDA path).

Run HERE (the build container), where the reference package is importable:

    python tests/golden/make_golden.py

It imports the reference ``seriesearch`` from /root/reference/pkg/src (read
only), runs the reference's own functions on small seeded inputs, and writes
``tests/golden/*.npz``.  The fixtures are committed; nothing on the GPU box
reads /root/reference.  Each block names the reference function that produced
it (paths relative to /root/reference/pkg/src/seriesearch).
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def random_walks(count: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    walks = np.cumsum(rng.standard_normal((count, n)), axis=1)
    mu = walks.mean(axis=1, keepdims=True)
    sd = walks.std(axis=1, keepdims=True)
    return ((walks - mu) / sd).astype(np.float32)


def main() -> None:
    sys.path.insert(0, REF)
    import seriesearch  # noqa: F401
    from seriesearch import core, generate, pscan, summarize, tree
    from seriesearch.build import build_index
    from seriesearch.persist import IndexSettings, write_index
    from seriesearch.query import QueryConfig, QueryEngine

    # -- core.py:50-57 ed2_batch -------------------------------------------
    ed = {}
    for n in (16, 64, 96, 256, 320):
        X = random_walks(40, n, 100 + n)
        q = random_walks(1, n, 200 + n)[0]
        ed[f"X{n}"] = X
        ed[f"q{n}"] = q
        ed[f"d2_{n}"] = core.ed2_batch(X, q)
    np.savez_compressed(os.path.join(OUT, "ed2.npz"), **ed)

    # -- pscan.py:23-30 brute_force_knn, with planted exact ties ------------
    X = random_walks(3000, 64, 7)
    X[2500] = X[10]          # duplicate rows -> exact distance ties
    X[2999] = X[10]
    X[1200] = X[1100]
    Q = np.concatenate([random_walks(6, 64, 8), X[[10, 1100]]])
    kn = {"X": X, "Q": Q}
    for k in (1, 10, 100):
        d2s, pos = [], []
        for q in Q:
            rs = pscan.brute_force_knn(X, q, k)
            d2s.append(rs.distances_sq())
            pos.append([p for _, p in rs.entries()])
        kn[f"d2_k{k}"] = np.array(d2s, np.float32)
        kn[f"id_k{k}"] = np.array(pos, np.int64)
    np.savez_compressed(os.path.join(OUT, "knn.npz"), **kn)

    # -- summarize.py:34-82 segment statistics --------------------------------
    st = {}
    X = random_walks(30, 256, 9)
    X[0, 5] = 1e4            # large magnitude: exercises the fp64 prefix path
    segs = {
        "root": ([0], [256]),
        "three": ([0, 16, 40], [16, 40, 256]),
        "fine": (list(range(0, 256, 7)), list(range(7, 256, 7)) + [256]),
        "width1": ([0, 1, 2, 200], [1, 2, 200, 256]),
    }
    st["X"] = X
    for name, (s, e) in segs.items():
        mean, sd = summarize.segment_stats_matrix(X, np.array(s), np.array(e))
        st[f"starts_{name}"] = np.array(s, np.int64)
        st[f"ends_{name}"] = np.array(e, np.int64)
        st[f"mean_{name}"] = mean
        st[f"sd_{name}"] = sd
    np.savez_compressed(os.path.join(OUT, "stats.npz"), **st)

    # -- summarize.py:89-133 PAA, breakpoints, SAX words ----------------------
    wd = {}
    bp = summarize.normal_breakpoints(256)
    wd["bp"] = bp
    lower, upper = summarize.symbol_bounds(bp)
    wd["lower"], wd["upper"] = lower, upper
    for n in (96, 256):
        X = random_walks(64, n, 300 + n)
        X[0, :] = 0.0                          # PAA exactly 0 -> tie to upper symbol
        X[1, : n // 16] = np.float32(bp[200])  # PAA on a breakpoint (as float32)
        p = summarize.paa_batch(X, 16)
        wd[f"X{n}"] = X
        wd[f"paa{n}"] = p
        wd[f"words{n}"] = summarize.isax_from_paa(p, bp)
    np.savez_compressed(os.path.join(OUT, "words.npz"), **wd)

    # -- summarize.py:136-153 lb_sax_batch -----------------------------------
    ls = {}
    n = 256
    data = random_walks(300, n, 11)
    queries = random_walks(5, n, 12)
    W = summarize.isax_from_paa(summarize.paa_batch(data, 16), bp)
    ls["W"] = W
    ls["qpaa"] = summarize.paa_batch(queries, 16)
    ls["lb"] = np.stack([summarize.lb_sax_batch(qp, W, lower, upper, n) for qp in ls["qpaa"]])
    ls["n"] = np.int64(n)
    np.savez_compressed(os.path.join(OUT, "lbsax.npz"), **ls)

    # -- summarize.py:170-206 lb_eapca / query.py:127-135 ---------------------
    le = {}
    rng = np.random.default_rng(13)
    data = random_walks(2000, 128, 14)
    qs = random_walks(12, 128, 15)
    cases = []
    for i, q in enumerate(qs):
        members = data[rng.choice(2000, size=40, replace=False)]
        cut = sorted(set(int(c) for c in rng.integers(1, 128, size=1 + i % 5)))
        endpoints = np.array(cut + [128], np.int64)
        starts = np.concatenate([[0], endpoints[:-1]])
        means, sds = summarize.segment_stats_matrix(members, starts, endpoints)
        env = [means.min(0), means.max(0), sds.min(0), sds.max(0)]
        lb = summarize.lb_eapca(q, endpoints, *env)
        le[f"q{i}"] = q
        le[f"ep{i}"] = endpoints
        for nm, v in zip(("mu_min", "mu_max", "sd_min", "sd_max"), env):
            le[f"{nm}{i}"] = v
        le[f"lb{i}"] = np.float64(lb)
        cases.append(i)
    le["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(OUT, "lbeapca.npz"), **le)

    # -- tree.py:240-336 get_best_split_policy --------------------------------
    sp = {}
    cases = []
    for c in range(10):
        n = (32, 64, 256)[c % 3]
        rho = (24, 65, 200)[c % 3]
        members = random_walks(rho, n, 500 + c)
        if c == 9:                        # identical members -> fallback policy
            members = np.tile(members[:1], (rho, 1))
        eps = [[n], [n // 2, n], [n // 4, n // 2, (3 * n) // 4, n]][c % 3]
        ids = tree.IdAllocator()
        leaf = tree.Node(ids.take(), eps)
        for s in members:
            tree.update_leaf_synopsis(leaf, s)
        pol = tree.get_best_split_policy(leaf, members)
        sp[f"members{c}"] = members
        sp[f"ep{c}"] = np.array(eps, np.int64)
        sp[f"mu_min0_{c}"] = np.float32(leaf.mu_min[0])
        sp[f"mu_max0_{c}"] = np.float32(leaf.mu_max[0])
        sp[f"pol{c}"] = np.array([pol.segment_index, 0 if pol.attribute == tree.MEAN else 1,
                                  -1 if pol.split_point is None else pol.split_point,
                                  pol.route_start, pol.route_end], np.int64)
        sp[f"thr{c}"] = np.float64(pol.threshold)
        sp[f"gain{c}"] = np.float64(pol.gain)
        sp[f"nleft{c}"] = np.int64(pol.route_mask(members).sum())
        cases.append(c)
    sp["count"] = np.int64(len(cases))
    np.savez_compressed(os.path.join(OUT, "split.npz"), **sp)

    # -- generate.py:27-81 seeded random walks and noisy queries --------------
    gn = {}
    gn["walk256_s0"] = generate.random_walk_block(0, 6, 256, 0)
    gn["walk256_s0_at1000"] = generate.random_walk_block(1000, 3, 256, 0)
    gn["walk96_s3"] = generate.random_walk_block(5, 4, 96, 3)
    base = generate.random_walk_block(0, 50, 64, 0)
    gn["noise_base"] = base
    for sigma in (0.01, 0.1, 1.0):
        qs = np.empty((5, 64), np.float32)
        srcs = np.empty(5, np.int64)
        for j in range(5):
            rng = generate._series_rng(1, j)
            src = int(rng.integers(len(base)))
            noisy = base[src].astype(np.float64) + rng.normal(0.0, sigma, 64)
            qs[j] = core.z_normalize(noisy.astype(np.float32))
            srcs[j] = src
        gn[f"noise_q_{sigma}"] = qs
        gn[f"noise_src_{sigma}"] = srcs
    np.savez_compressed(os.path.join(OUT, "generate.npz"), **gn)

    # -- the reference engine end to end (build_index/write_index/exact_knn) --
    en = {}
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "d.bin")
        generate.generate_random_walk(1500, 64, 11, path)
        settings = IndexSettings(series_length=64, dataset_size=1500, leaf_threshold=64)
        idx = build_index(path, settings, num_threads=2)
        idx_dir = os.path.join(OUT, "ref_index_1500x64")
        import shutil
        shutil.rmtree(idx_dir, ignore_errors=True)
        qidx = write_index(idx, idx_dir, num_threads=1)
        data = core.read_series_file(path, 64)
        queries = np.concatenate([generate.random_walk_block(0, 4, 64, 1),
                                  data[[3, 700]] + np.float32(0.01)])
        eng = QueryEngine(qidx)
        for k in (1, 10):
            d2s = []
            for q in queries:
                rs, _ = eng.exact_knn(q, QueryConfig(k=k))
                d2s.append(rs.distances_sq())
            en[f"d2_k{k}"] = np.array(d2s, np.float32)
        eng.close()
        en["data"] = data
        en["queries"] = queries.astype(np.float32)
        en["leaves"] = np.int64(qidx.total_leaves)
    np.savez_compressed(os.path.join(OUT, "engine.npz"), **en)
    print("wrote", sorted(f for f in os.listdir(OUT) if f.endswith(".npz")))


if __name__ == "__main__":
    main()
