"""Randomised parity stress of the projected tensor-core filter (K-proj: alternating epilogue
groups, candidate queue) and of auto routing against the oracle: random index sizes, series
lengths, noise levels and k (GPU box).

    python tools/proj_stress.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402  (the checker)
import paper_2212_13297_b200 as ssb  # noqa: E402

rng = np.random.default_rng(321)
bad = 0
cases = 0
for it in range(10):
    n = int(rng.choice([128, 256]))
    N = int(rng.integers(150_000, 900_000))
    X = np.cumsum(rng.standard_normal((N, n), dtype=np.float32), axis=1)
    X = ((X - X.mean(1, keepdims=True)) / X.std(1, keepdims=True)).astype(np.float32)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=n, dataset_size=N, leaf_threshold=int(rng.choice([2000, 10000]))))
    eng = ssb.QueryEngine(idx)
    B = int(rng.integers(33, 300))
    sigma = float(rng.choice([0.01, 0.1, 1.0]))
    Q = X[rng.integers(0, N, B)] + np.float32(sigma) * rng.standard_normal((B, n)).astype(np.float32)
    Q = ((Q - Q.mean(1, keepdims=True)) / Q.std(1, keepdims=True)).astype(np.float32)
    for k in (1, 10, 100):
        od2, oid = oracle.knn_scan(X, Q, k, threads=16)
        for route in ("proj", "auto"):
            d2, ids, _ = eng.knn_device(Q, k, route=route)
            ok = np.array_equal(ids.cpu().numpy(), oid) and np.array_equal(d2.cpu().numpy().view(np.uint32), od2.view(np.uint32))
            cases += 1
            if not ok:
                bad += 1
                print("MISMATCH", it, n, N, B, sigma, k, route)
    del eng, idx
print(f"proj stress: {cases} cases, {bad} mismatches")
