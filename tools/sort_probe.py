"""Does ordering the queries of a call by their best leaf (LB_EAPCA) speed up
the tensor-core filter?  (GPU box; C2 shape)"""
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

    N, n = 1_000_000, 256
    X = G.random_walks(N, n, 0)
    idx = ssb.build_index_array(torch.from_numpy(X).cuda(), ssb.IndexSettings(series_length=n, dataset_size=N,
                                                                               leaf_threshold=10_000))
    L = idx.info.num_leaves
    eng = ssb.QueryEngine(idx)
    Q = np.concatenate([G.noise_queries(X, 1000, s, 1) for s in (0.01, 0.1, 1.0)])
    Qd = torch.from_numpy(Q).cuda()
    lbe = torch.empty((len(Q), L), dtype=torch.float64, device="cuda")
    _lib.call("ssb_index_lb_eapca", idx.handle, ctypes.c_void_p(Qd.data_ptr()), len(Q),
              ctypes.c_void_p(lbe.data_ptr()), None)
    best = lbe.argmin(1).cpu().numpy()
    order = np.argsort(best, kind="stable")
    rnd = np.random.default_rng(5).permutation(len(Q))
    for name, QQ in (("as-is", Qd), ("by-best-leaf", Qd[torch.from_numpy(order).cuda()].contiguous()),
                     ("shuffled", Qd[torch.from_numpy(rnd).cuda()].contiguous())):
        for k in (1, 10):
            eng.knn_device(QQ, k)
            torch.cuda.synchronize()
            _lib.prof_reset()
            _lib.prof_enable(True)
            eng.knn_device(QQ, k)
            torch.cuda.synchronize()
            _lib.prof_enable(False)
            prof = _lib.prof_read()
            print(json.dumps({"order": name, "k": k, "kernels": {kk: round(v[0], 3) for kk, v in prof.items()}}))


if __name__ == "__main__":
    main()
