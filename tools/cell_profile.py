"""Per-cell profile of the C2 workload on the index engine (GPU box).

    python tools/cell_profile.py [--rows N] [--queries Q] [--tau T]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--tau", type=int, default=10_000)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--sigmas", default="0.01,0.1,1.0")
    ap.add_argument("--ks", default="1,10")
    a = ap.parse_args()
    import torch

    import paper_2212_13297_b200 as ssb
    from paper_2212_13297_b200 import _lib
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(a.rows, a.n, 0)
    Xd = torch.from_numpy(X).cuda()
    s = ssb.IndexSettings(series_length=a.n, dataset_size=a.rows, leaf_threshold=a.tau)
    t0 = time.perf_counter()
    idx = ssb.build_index_array(Xd, s)
    torch.cuda.synchronize()
    print(json.dumps({"build_s": round(time.perf_counter() - t0, 3), "leaves": idx.info.num_leaves}))
    eng = ssb.QueryEngine(idx)
    for sigma in [float(v) for v in a.sigmas.split(",")]:
        Q = torch.from_numpy(G.noise_queries(X, a.queries, sigma, 1)).cuda()
        for k in [int(v) for v in a.ks.split(",")]:
            eng.knn_device(Q, k)  # warm
            torch.cuda.synchronize()
            _lib.prof_reset()
            _lib.prof_enable(True)
            t0 = time.perf_counter()
            d2, ids, pos, st = eng.knn_device(Q, k, want_stats=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            _lib.prof_enable(False)
            prof = _lib.prof_read()
            print(json.dumps({
                "sigma": sigma, "k": k, "ms": round(1000 * dt, 2),
                "cand_leaves": float(st[:, 0].mean()), "cand_series": float(st[:, 1].mean()),
                "seed_rows": float(st[:, 2].mean()), "overflowed": int(st[:, 3].sum()),
                "kernels": {kk: [round(v[0], 3), v[1], round(v[2] / 1e9, 3)] for kk, v in prof.items()}}))


if __name__ == "__main__":
    main()
