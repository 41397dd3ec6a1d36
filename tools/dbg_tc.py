import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/oracle')
from conftest import random_walks
import oracle
import paper_2212_13297_b200 as ssb
for N, k in [(70, 100), (70, 40), (70, 20), (200, 100), (300, 64)]:
    X = random_walks(N, 64, 9)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=64, dataset_size=N, leaf_threshold=4))
    Q = random_walks(3, 64, 10)
    od2, oid = oracle.knn_scan(X, Q, k)
    for route in ("tensor", "tree"):
        d2, ids, _, st = ssb.QueryEngine(idx).knn_device(Q, k, want_stats=True, route=route)
        ok = np.array_equal(ids.cpu().numpy(), oid)
        print(N, k, route, ok, st[:, 1].tolist())
