"""How much of the dense tensor-core scan could the index skip? (GPU box)

For each C2 sigma: per query, the leaves whose LB_EAPCA does not exceed the
final k-th distance (those the exact answer needs); queries sorted by their best
leaf and grouped in blocks of 128; per block, the fraction of rows in leaves
some query of the block needs.
"""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2212_13297_b200 as ssb
    from paper_2212_13297_b200 import _lib
    from paper_2212_13297_b200 import generate as G

    N, n, tau = 1_000_000, 256, 10_000
    X = G.random_walks(N, n, 0)
    idx = ssb.build_index_array(torch.from_numpy(X).cuda(),
                                ssb.IndexSettings(series_length=n, dataset_size=N, leaf_threshold=tau))
    leaves = idx.leaves_inorder()
    counts = np.array([l.file_position[1] for l in leaves], np.int64)
    L = len(leaves)
    eng = ssb.QueryEngine(idx)
    for sigma in (0.01, 0.1, 1.0):
        Q = G.noise_queries(X, 1000, sigma, 1)
        Qd = torch.from_numpy(Q).cuda()
        for k in (1, 10):
            d2, ids, _ = eng.knn_device(Qd, k)
            kth = d2[:, -1].double().cpu().numpy()
            lbe = torch.empty((len(Q), L), dtype=torch.float64, device="cuda")
            _lib.call("ssb_index_lb_eapca", idx.handle, ctypes.c_void_p(Qd.data_ptr()), len(Q),
                      ctypes.c_void_p(lbe.data_ptr()), None)
            lb = lbe.cpu().numpy()
            need = lb <= kth[:, None] * (1 + 1e-5) + 1e-6
            per_q = (need * counts[None, :]).sum(1) / N
            best = lb.argmin(1)
            order = np.argsort(best, kind="stable")
            fr = []
            for b0 in range(0, len(Q), 128):
                blk = order[b0:b0 + 128]
                u = need[blk].any(0)
                fr.append((u * counts).sum() / N)
            print(json.dumps({"sigma": sigma, "k": k, "rows_needed_per_query": round(float(per_q.mean()), 4),
                              "rows_needed_per_sorted_block": round(float(np.mean(fr)), 4),
                              "unsorted_block": round(float(np.mean([(need[b0:b0 + 128].any(0) * counts).sum() / N
                                                                    for b0 in range(0, len(Q), 128)])), 4)}))


if __name__ == "__main__":
    main()
