"""Per-kernel profile of the level-synchronous index build (GPU box).

    python tools/build_profile.py [--rows N] [--n 256] [--tau T]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--tau", type=int, default=10_000)
    ap.add_argument("--no-warm", action="store_true", help="skip the small warm-up build (profilers)")
    ap.add_argument("--repeat", type=int, default=1, help="timed builds (the profile covers the last)")
    a = ap.parse_args()
    import torch

    import paper_2212_13297_b200 as ssb
    from paper_2212_13297_b200 import _lib
    from paper_2212_13297_b200 import generate as G

    X = torch.from_numpy(G.random_walks(a.rows, a.n, 0)).cuda()
    s = ssb.IndexSettings(series_length=a.n, dataset_size=a.rows, leaf_threshold=a.tau)
    if not a.no_warm:  # module loading and pool growth outside the measured build
        w = min(a.rows, 200_000)
        ssb.build_index_array(X[:w], ssb.IndexSettings(series_length=a.n, dataset_size=w, leaf_threshold=a.tau))
    torch.cuda.synchronize()
    walls = []
    for _ in range(a.repeat):
        idx = None
        _lib.prof_reset()
        _lib.prof_enable(True)
        t0 = time.perf_counter()
        idx = ssb.build_index_array(X, s)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        walls.append(round(dt, 4))
    _lib.prof_enable(False)
    prof = _lib.prof_read()
    print(json.dumps({"rows": a.rows, "s": round(dt, 3), "series_per_s": round(a.rows / dt),
                      "levels": idx.info.levels, "leaves": idx.info.num_leaves, "walls": walls,
                      "kernels": {k: [round(v[0], 2), v[1], round(v[2] / 1e9, 2)] for k, v in prof.items()}}))


if __name__ == "__main__":
    main()
