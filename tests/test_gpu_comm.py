"""The library's row-shard communicator (csrc/comm.cu) on one
GPU: a one-rank NCCL communicator through the C ABI.  The merge of one shard
is the shard's own answer; an index with the communicator attached (bound
all-reduce, rank-independent routing) answers exactly like the oracle.  (The
multi-rank data path runs under bench.py --gpus N; its host logic is covered
by the gloo tests in test_distributed_cpu.py.)"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
THREADS = os.cpu_count() or 8


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def test_one_rank_comm_merge_and_bounds(oracle):
    import torch

    import paper_2212_13297_b200 as ssb
    from paper_2212_13297_b200 import generate as G
    from paper_2212_13297_b200.distributed import Comm

    X = G.random_walks(120_000, 256, 21)
    Q = G.noise_queries(X, 48, 0.1, 22)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=2000))
    eng = ssb.QueryEngine(idx)
    comm = Comm(0, 1)
    try:
        for k in (1, 10, 100):
            d2, ids, _ = eng.knn_device(Q, k)
            md2, mids = comm.merge(d2, ids, k)
            assert torch.equal(mids, ids) and torch.equal(md2, d2)
        comm.attach(idx)
        od2, oid = oracle.knn_scan(X, Q, 10, threads=THREADS)
        for route in ("auto", "proj", "tree"):
            d2, ids, _ = eng.knn_device(Q, 10, route=route)
            assert np.array_equal(ids.cpu().numpy(), oid), route
            assert np.array_equal(bits(d2.cpu().numpy()), bits(od2)), route
        rs, _ = eng.exact_knn(Q[0], ssb.QueryConfig(k=10))  # a single query: no graph replay with a comm
        assert rs.ids() == list(oid[0])
    finally:
        comm.close()


def test_merge_pads_empty_slots():
    """k larger than a shard: empty slots stay (inf, -1) through the merge."""
    import torch

    from paper_2212_13297_b200.distributed import Comm

    comm = Comm(0, 1)
    try:
        d2 = torch.tensor([[1.0, 2.0, float("inf")]], device="cuda")
        ids = torch.tensor([[5, 3, -1]], dtype=torch.int64, device="cuda")
        md2, mids = comm.merge(d2, ids, 3)
        assert mids.cpu().tolist() == [[5, 3, -1]]
        assert md2[0, 2].item() == float("inf")
    finally:
        comm.close()
