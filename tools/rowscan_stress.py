"""Randomised parity stress of ssb_bruteforce_knn for B <= 4 (the streamed exact row scan) against
the oracle: random n / N / B / k, near-duplicate, far and exact-duplicate queries (GPU box).

    python tools/rowscan_stress.py
"""
import sys, os
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle
import paper_2212_13297_b200 as ssb
rng = np.random.default_rng(123)
bad = 0
for it in range(60):
    n = int(rng.choice([64, 96, 128, 256]))
    N = int(rng.integers(1, 150_000))
    B = int(rng.integers(1, 5))
    k = int(rng.choice([1, 2, 7, 10, 33, 100, 256]))
    X = np.cumsum(rng.standard_normal((N, n)), axis=1)
    X = ((X - X.mean(1, keepdims=True)) / (X.std(1, keepdims=True) + 1e-9)).astype(np.float32)
    kind = it % 3
    if kind == 0:
        Q = X[rng.integers(0, N, B)] + np.float32(0.05) * rng.standard_normal((B, n)).astype(np.float32)
    elif kind == 1:
        Q = rng.standard_normal((B, n)).astype(np.float32) * np.float32(rng.choice([0.1, 1.0, 30.0]))
    else:
        Q = X[rng.integers(0, N, B)].copy()  # exact duplicates present
        dup = rng.integers(0, N, 5)
        X[dup] = Q[0]
    Q = Q.astype(np.float32)
    d2, ids = ssb.knn_batch(X, Q, k)
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    ok = np.array_equal(ids.cpu().numpy(), oid) and np.array_equal(d2.cpu().numpy().view(np.uint32), od2.view(np.uint32))
    if not ok:
        bad += 1
        print("MISMATCH", it, n, N, B, k, kind)
print("rowscan stress: 60 cases,", bad, "mismatches")
