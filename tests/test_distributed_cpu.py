"""Multi-process (gloo, world_size 2) test of the row-sharded path's host
logic: shard ranges, global ids, the all-gather and the (d2, id) merge.  The
per-shard search is the oracle (no GPU here); the product path uses the same
plumbing with the device search and the K-merge kernel."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import random_walks


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _host_merge(all_keys, k):
    from paper_2212_13297_b200.distributed import host_merge

    return host_merge(all_keys, k)


def _worker(rank, world, port, X, Q, k, out):
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import oracle

    from paper_2212_13297_b200.distributed import merge_topk, shard_range

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(len(X), rank, world)
    d2, ids = oracle.knn_scan(X[lo:hi], Q, k)
    ids = np.where(ids >= 0, ids + lo, -1)  # global ids (id_base = lo)
    gd2, gids = merge_topk(torch.from_numpy(d2), torch.from_numpy(ids), k, merge_fn=_host_merge)
    if rank == 0:
        out.put((np.asarray(gd2), np.asarray(gids)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_merge_equals_global_scan(oracle, world):
    X = random_walks(3001, 64, 21)
    X[2999] = X[5]            # a tie across shards: the lowest global id must win
    Q = np.concatenate([random_walks(5, 64, 22), X[[5]]])
    k = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, Q, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    gd2, gids = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    od2, oid = oracle.knn_scan(X, Q, k)
    assert np.array_equal(gids, oid)
    assert np.array_equal(gd2.view(np.uint32), od2.view(np.uint32))
    assert list(gids[-1][:2]) == [5, 2999]


def test_shard_ranges_cover_and_pack_roundtrip():
    from paper_2212_13297_b200.distributed import pack_keys, shard_range, unpack_keys

    for N in (1, 7, 1000, 25_000_000):
        for world in (1, 2, 3, 8):
            r = [shard_range(N, i, world) for i in range(world)]
            assert r[0][0] == 0 and r[-1][1] == N
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    d2 = np.array([[0.0, 1.5, np.inf]], np.float32)
    ids = np.array([[3, 2**31 + 5, -1]], np.int64)
    back = unpack_keys(pack_keys(d2, ids))
    assert np.array_equal(back[0], d2) and np.array_equal(back[1], ids)
    # empty slots are all-ones keys (the K-merge kernel's KEY_EMPTY) and sort last
    keys = pack_keys(d2, ids)
    assert keys[0, 2] == -1 and keys.view(np.uint64)[0, 2] == np.uint64(2**64 - 1)


def test_host_merge_pads_k_above_n():
    """k > total rows: missing answers come back as (inf, -1), like query.py:70-75."""
    import torch

    from paper_2212_13297_b200.distributed import host_merge, pack_keys

    a = pack_keys(np.array([[1.0, np.inf]], np.float32), np.array([[4, -1]], np.int64))
    b = pack_keys(np.array([[0.5, np.inf]], np.float32), np.array([[9, -1]], np.int64))
    d2, ids = host_merge(torch.from_numpy(np.concatenate([a, b], axis=1)), 5)
    assert list(ids[0]) == [9, 4, -1, -1, -1]
    assert d2[0, 0] == np.float32(0.5) and np.isinf(d2[0, 2:]).all()
