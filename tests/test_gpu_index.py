"""Index build (K-split/K-part) and pruned exact query (K-lbe/K-lbs/K-scan/
K-select) on the B200, checked against the oracle and reference goldens.

Bars: ids identical to the oracle's full scan (ties -> lowest index), squared
distances bit-identical; every split policy identical to the reference's
get_best_split_policy on the node's split set -- the members the reference's
sequential insertion build splits on (build.py:213-263): the node's first
max(inherited + 1, tau + 1) members in original order -- (threshold and gain
bit-equal); the whole tree identical to a reference-built index; envelopes
bit-equal to min/max of the members' statistics; words bit-equal.
"""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden, random_walks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ssb():
    import paper_2212_13297_b200 as ssb

    return ssb


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def build(ssb, X, tau, **kw):
    s = ssb.IndexSettings(series_length=X.shape[1], dataset_size=X.shape[0], leaf_threshold=tau)
    return ssb.build_index_array(X, s, **kw)


def noisy(X, count, sigma, seed):
    rng = np.random.default_rng(seed)
    out = np.empty((count, X.shape[1]), np.float32)
    for i, src in enumerate(rng.integers(0, len(X), size=count)):
        v = X[src].astype(np.float64) + rng.normal(0, sigma, X.shape[1])
        out[i] = ((v - v.mean()) / v.std()).astype(np.float32)
    return out


@pytest.fixture(scope="module")
def small(ssb):
    X = random_walks(2000, 64, 11)
    return X, build(ssb, X, 64)


def check_tree(ssb, oracle, X, idx, tau, max_policy_checks=10_000):
    rows, words, ids = idx.host_arrays()
    N, n = X.shape
    # multiset / permutation: every series exactly once, rows moved intact
    assert sorted(ids.tolist()) == list(range(N))
    assert np.array_equal(rows, X[ids])
    # words of the leaf-ordered rows
    bp = oracle.normal_breakpoints(256)
    assert np.array_equal(words, oracle.words(rows, bp))
    checked = 0
    leaves = list(idx.root.iter_leaves())
    pos = 0
    for leaf in leaves:
        first, count = leaf.file_position
        assert first == pos
        pos += count
        assert count <= tau or leaf.oversize or count == leaf.inherited
    assert pos == N
    for node in idx.root.iter_nodes():
        first, count = node.file_position
        members = rows[first:first + count]
        mean, sd = oracle.segment_stats(members, node.starts, node.endpoints)
        # exact envelopes (tree.py:143-155 over the node's own members)
        assert np.array_equal(bits(node.mu_min), bits(mean.min(0)))
        assert np.array_equal(bits(node.mu_max), bits(mean.max(0)))
        assert np.array_equal(bits(node.sd_min), bits(sd.min(0)))
        assert np.array_equal(bits(node.sd_max), bits(sd.max(0)))
        if not node.is_leaf and checked < max_policy_checks:
            S = node.split_set
            assert S == max(node.inherited + 1, tau + 1) and S <= count
            split_set = X[np.sort(ids[first:first + count])[:S]]
            smean, _ = oracle.segment_stats(split_set, node.starts, node.endpoints)
            pol = oracle.best_split(split_set, node.endpoints, float(smean[:, 0].min()),
                                    float(smean[:, 0].max()),
                                    allow_vsplit=node.num_segments < 32)
            p = node.policy
            assert (p.segment_index, p.attribute, p.split_point, p.route_start, p.route_end) == (
                pol["segment_index"], pol["attribute"], pol["split_point"], pol["route_start"],
                pol["route_end"]), node
            assert p.threshold == pol["threshold"]
            assert p.gain == pol["gain"]
            assert node.left.inherited == pol["n_left"]
            assert node.right.inherited == S - pol["n_left"]
            assert node.left.file_position[1] + node.right.file_position[1] == count
            checked += 1
    return checked


def test_build_small_matches_reference_policies(ssb, oracle, small):
    X, idx = small
    assert idx.info.num_leaves > 10
    checked = check_tree(ssb, oracle, X, idx, 64)
    assert checked == idx.info.num_nodes - idx.info.num_leaves


@pytest.mark.parametrize("n,N,tau,seed", [(256, 20_000, 1000, 1), (96, 12_000, 500, 2),
                                          (128, 3_001, 100, 3)])
def test_build_matches_reference_policies(ssb, oracle, n, N, tau, seed):
    X = random_walks(N, n, seed)
    idx = build(ssb, X, tau)
    check_tree(ssb, oracle, X, idx, tau, max_policy_checks=60)


def test_build_edges(ssb, oracle):
    X = random_walks(50, 64, 4)
    idx = build(ssb, X, 100)                       # tau >= N: the root is the only leaf
    assert idx.info.num_leaves == 1 and idx.root.is_leaf
    check_tree(ssb, oracle, X, idx, 100)
    one = build(ssb, X[:1], 1)                     # a single series
    assert one.info.num_leaves == 1
    dup = np.tile(X[:1], (40, 1))                  # identical members: cannot split
    d = build(ssb, dup, 4)
    assert d.info.num_leaves == 1 and d.root.oversize
    mixed = np.concatenate([dup, X[1:30]])         # duplicates plus distinct rows
    m = build(ssb, mixed, 4)
    check_tree(ssb, oracle, mixed, m, 4)
    with pytest.raises(ssb.UsageError):
        bad = X.copy()
        bad[3, 7] = np.nan
        build(ssb, bad, 10)
    init = build(ssb, X, 8, initial_segments=16)   # config 1's "16 initial segments"
    assert init.root.num_segments == 16
    check_tree(ssb, oracle, X, init, 8)


@pytest.mark.parametrize("k", [1, 10, 100])
def test_query_equals_oracle_scan(ssb, oracle, small, k):
    X, idx = small
    Q = np.concatenate([noisy(X, 12, 0.3, 31), random_walks(6, 64, 32), X[[5, 1999]]])
    d2, ids, pos = ssb.QueryEngine(idx).knn_device(Q, k)
    od2, oid = oracle.knn_scan(X, Q, k)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2))
    rows, _, orig = idx.host_arrays()
    p = pos.cpu().numpy()
    valid = p >= 0
    assert np.array_equal(orig[p[valid]], ids.cpu().numpy()[valid])


@pytest.mark.parametrize("sigma", [0.01, 0.1, 1.0])
@pytest.mark.parametrize("k", [1, 10])
def test_query_c2_shape_small(ssb, oracle, sigma, k):
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(30_000, 256, 0, workers=4)
    idx = build(ssb, X, 1000)
    Q = G.noise_queries(X, 64, sigma, 1)
    eng = ssb.QueryEngine(idx)
    od2, oid = oracle.knn_scan(X, Q, k, threads=8)
    for route in ("tree", "auto"):
        d2, ids, pos, st = eng.knn_device(Q, k, want_stats=True, route=route)
        assert np.array_equal(ids.cpu().numpy(), oid), route
        assert np.array_equal(bits(d2.cpu().numpy()), bits(od2)), route
        if sigma <= 0.1:   # the filters must actually filter on easy queries
            assert st[:, 1].mean() < 0.2 * len(X), route


def test_query_ties_and_duplicates(ssb, oracle):
    X = random_walks(3000, 64, 7)
    X[2500] = X[10]
    X[2999] = X[10]
    X[1200] = X[1100]
    idx = build(ssb, X, 50)
    Q = X[[10, 1100]]
    d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, 3)
    ids = ids.cpu().numpy()
    assert list(ids[0]) == [10, 2500, 2999]
    assert list(ids[1][:2]) == [1100, 1200]


def test_query_k_larger_than_n_and_tiny_leaves(ssb, oracle):
    X = random_walks(70, 64, 9)
    idx = build(ssb, X, 4)
    Q = random_walks(3, 64, 10)
    d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, 100)
    od2, oid = oracle.knn_scan(X, Q, 100)
    assert np.array_equal(ids.cpu().numpy(), oid)
    assert (ids.cpu().numpy()[:, 70:] == -1).all()


def test_query_overflow_tightening(ssb, oracle):
    # tau > candidate capacity and wide-open bounds force the K-select
    # overflow -> tighter-bound -> rescan loop
    X = random_walks(60_000, 64, 12)
    idx = build(ssb, X, 40_000)
    Q = random_walks(4, 64, 13)
    d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, 20)
    od2, oid = oracle.knn_scan(X, Q, 20, threads=8)
    assert np.array_equal(ids.cpu().numpy(), oid)


def test_engine_matches_reference_engine_golden(ssb):
    g = golden("engine")
    X = g["data"]
    idx = build(ssb, X, 64)
    eng = ssb.QueryEngine(idx)
    for k in (1, 10):
        res = eng.exact_knn_batch(g["queries"], ssb.QueryConfig(k=k))
        got = np.array([r.distances_sq() for r, _ in res], np.float32)
        assert np.array_equal(bits(got), bits(g[f"d2_k{k}"])), k


def test_build_reproduces_reference_built_tree(ssb):
    """The reference's build_index (one insert worker: sequential insertion in
    file order) wrote tests/golden/ref_index_1500x64 from the same 1500 series;
    the level-synchronous GPU build must give the same tree: node by node the
    same structure, segmentations, policies (threshold bits) and envelopes, and
    leaf by leaf the same series in the same order."""
    g = golden("engine")
    qi = ssb.load_index(os.path.join(GOLDEN, "ref_index_1500x64"))
    ours = build(ssb, g["data"], 64)
    rows, _, _ = ours.host_arrays()
    ref_rows = qi.store.data

    def walk(a, b, path="root"):
        assert a.is_leaf == b.is_leaf, path
        assert np.array_equal(a.endpoints, b.endpoints), path
        for f in ("mu_min", "mu_max", "sd_min", "sd_max"):
            assert np.array_equal(bits(getattr(a, f)), bits(getattr(b, f))), (path, f)
        fa, ca = a.file_position
        fb, cb = b.file_position
        assert ca == cb, path
        if a.is_leaf:
            assert np.array_equal(rows[fa:fa + ca], ref_rows[fb:fb + cb]), path
            return 1
        pa, pb = a.policy, b.policy
        assert (pa.segment_index, pa.attribute, pa.split_point, pa.route_start, pa.route_end) == (
            pb.segment_index, pb.attribute, pb.split_point, pb.route_start, pb.route_end), path
        assert pa.threshold == pb.threshold, path
        return walk(a.left, b.left, path + "L") + walk(a.right, b.right, path + "R")

    assert walk(ours.root, qi.root) == qi.total_leaves


def test_reference_written_index_loads_and_answers(ssb, oracle):
    g = golden("engine")
    qi = ssb.load_index(os.path.join(GOLDEN, "ref_index_1500x64"))
    assert qi.total_leaves == int(g["leaves"])
    eng = ssb.QueryEngine(qi)
    rows = qi.store.data
    for k in (1, 10):
        d2, ids, pos = eng.knn_device(g["queries"], k)
        od2, oid = oracle.knn_scan(rows, g["queries"], k)
        assert np.array_equal(ids.cpu().numpy(), oid)   # positions stand in for ids
        assert np.array_equal(bits(d2.cpu().numpy()), bits(g[f"d2_k{k}"]))


def test_write_then_load_round_trip(ssb, oracle, small, tmp_path):
    X, idx = small
    qi = ssb.write_index(idx, str(tmp_path / "ix"))
    back = ssb.load_index(str(tmp_path / "ix"))
    assert back.total_leaves == qi.total_leaves
    Q = noisy(X, 8, 0.2, 40)
    a = ssb.QueryEngine(qi).knn_device(Q, 5)
    b = ssb.QueryEngine(back).knn_device(Q, 5)
    for u, v in zip(a, b):
        assert np.array_equal(u.cpu().numpy(), v.cpu().numpy())
    with open(tmp_path / "ix" / "htree.bin", "r+b") as f:
        f.write(b"XXXXXXXX")
    with pytest.raises(ssb.IntegrityError):
        ssb.load_index(str(tmp_path / "ix"))


def test_lb_eapca_bitwise_vs_oracle(ssb, oracle, small):
    import ctypes

    import torch

    from paper_2212_13297_b200 import _lib

    X, idx = small
    Q = noisy(X, 5, 0.5, 41)
    leaves = list(idx.root.iter_leaves())
    out = torch.empty((5, len(leaves)), dtype=torch.float64, device="cuda")
    q = torch.from_numpy(Q).cuda()
    _lib.call("ssb_index_lb_eapca", idx.handle, ctypes.c_void_p(q.data_ptr()), 5,
              ctypes.c_void_p(out.data_ptr()), None)
    out = out.cpu().numpy()
    for i in range(5):
        for j, leaf in enumerate(leaves):
            ref = oracle.lb_eapca_query(Q[i], leaf.endpoints, leaf.mu_min, leaf.mu_max, leaf.sd_min,
                                        leaf.sd_max)
            assert out[i, j] == ref


def test_lb_sax_bitwise_vs_golden(ssb):
    import ctypes

    import torch

    from paper_2212_13297_b200 import _lib

    g = golden("lbsax")
    lo, hi = (torch.from_numpy(v).cuda() for v in ssb.summarize.symbol_bounds(
        ssb.summarize.normal_breakpoints(256)))
    W = torch.from_numpy(np.ascontiguousarray(g["W"])).cuda()
    for i, qp in enumerate(g["qpaa"]):
        q = torch.from_numpy(np.ascontiguousarray(qp)).cuda()
        out = torch.empty(W.shape[0], dtype=torch.float64, device="cuda")
        _lib.call("ssb_lb_sax", ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(W.data_ptr()),
                  W.shape[0], ctypes.c_void_p(lo.data_ptr()), ctypes.c_void_p(hi.data_ptr()),
                  int(g["n"]), ctypes.c_void_p(out.data_ptr()), None)
        assert np.array_equal(out.cpu().numpy(), g["lb"][i])


def test_api_surface_and_errors(ssb, small, tmp_path):
    X, idx = small
    eng = ssb.QueryEngine(idx)
    rs, st = eng.exact_knn(X[3], ssb.QueryConfig(k=2))
    assert rs.entries()[0] == (0.0, rs.positions()[0]) and rs.ids()[0] == 3
    assert 0.0 <= st.fraction_data_accessed <= 1.0 and st.phase_reached in {"scan2", "scan3", "4", "3", "1"}
    with pytest.raises(ssb.UsageError):
        eng.exact_knn(np.zeros(7, np.float32), ssb.QueryConfig(k=1))
    with pytest.raises(ssb.UsageError):
        eng.exact_knn(X[0], ssb.QueryConfig(k=0))
    bad = X[0].copy()
    bad[0] = np.inf
    with pytest.raises(ssb.UsageError):
        eng.exact_knn(bad, ssb.QueryConfig(k=1))
    path = str(tmp_path / "d.bin")
    X.tofile(path)
    s = ssb.IndexSettings(series_length=64, dataset_size=2000, leaf_threshold=64)
    with pytest.raises(ssb.UsageError):
        ssb.build_index(path, s, num_threads=1)
    b = ssb.build_index(path, s, num_threads=2)
    assert b.info.num_leaves == idx.info.num_leaves


def test_sharded_forest_merge_on_device(ssb, oracle):
    """Row shards as separate device indexes + the K-merge kernel: the answer
    equals one global scan (multi-GPU data path, emulated on one GPU without
    any rank waiting on another)."""
    import torch

    from paper_2212_13297_b200.distributed import merge_device, pack_keys, shard_range

    X = random_walks(9000, 64, 31)
    X[8500] = X[7]
    Q = np.concatenate([noisy(X, 10, 0.3, 32), X[[7]]])
    k = 10
    world = 3
    parts = []
    for r in range(world):
        lo, hi = shard_range(len(X), r, world)
        s = ssb.IndexSettings(series_length=64, dataset_size=hi - lo, leaf_threshold=200)
        idx = ssb.build_index_array(X[lo:hi], s, id_base=lo)
        d2, ids, _ = ssb.QueryEngine(idx).knn_device(Q, k)
        parts.append(pack_keys(d2, ids))
    all_keys = torch.stack(parts).permute(1, 0, 2).reshape(len(Q), world * k).contiguous()
    gd2, gids = merge_device(all_keys, k)
    od2, oid = oracle.knn_scan(X, Q, k)
    assert np.array_equal(gids.cpu().numpy(), oid)
    assert np.array_equal(bits(gd2.cpu().numpy()), bits(od2))
    assert list(gids.cpu().numpy()[-1][:2]) == [7, 8500]


def test_device_merge_pads_k_above_total(ssb, oracle):
    """Shards holding fewer than k rows in total: the device packing marks the
    missing answers as empty keys and the K-merge returns (inf, -1) for them,
    like query.py:70-75."""
    import torch

    from paper_2212_13297_b200.distributed import merge_device, pack_keys

    X = random_walks(7, 64, 33)
    Q = X[[2, 5]]
    k = 10
    parts = []
    for lo, hi in ((0, 3), (3, 7)):
        d2, ids = ssb.knn_batch(X[lo:hi], Q, k, id_base=lo)
        keys = pack_keys(d2, ids)
        assert keys.is_cuda and (keys[:, hi - lo:] == -1).all()
        parts.append(keys)
    all_keys = torch.cat(parts, dim=1).contiguous()
    gd2, gids = merge_device(all_keys, k)
    od2, oid = oracle.knn_scan(X, Q, k)
    assert np.array_equal(gids.cpu().numpy(), oid)
    assert (gids.cpu().numpy()[:, 7:] == -1).all() and np.isinf(gd2.cpu().numpy()[:, 7:]).all()
    assert np.array_equal(bits(gd2.cpu().numpy()[:, :7]), bits(od2[:, :7]))


def test_small_blocks_cuda_graph_path(ssb, oracle):
    """Blocks of <= 64 queries on the index route replay a captured CUDA graph
    (one per stream, B, k, lmax); repeated calls, different k / lmax / block
    sizes and the per-query API all give the oracle's answers, with stats."""
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(60_000, 256, 3, workers=4)
    idx = ssb.build_index_array(X, ssb.IndexSettings(series_length=256, dataset_size=len(X), leaf_threshold=2000))
    eng = ssb.QueryEngine(idx)
    Q = np.concatenate([G.noise_queries(X, 12, 0.05, 4), G.random_walks(4, 256, 5, workers=1)])
    for k in (1, 10, 100):
        od2, oid = oracle.knn_scan(X, Q, k, threads=8)
        for B in (1, 3, 16):
            for rep in range(2):  # capture, then replay
                for q0 in range(0, len(Q), B):
                    d2, ids, _, st = eng.knn_device(Q[q0:q0 + B], k, want_stats=True)
                    assert np.array_equal(ids.cpu().numpy(), oid[q0:q0 + B]), (k, B, q0)
                    assert np.array_equal(bits(d2.cpu().numpy()), bits(od2[q0:q0 + B])), (k, B, q0)
                    if B <= 3:  # the graph-replayed blocks take the index route
                        assert (st[:, 7] == 0).all() and (st[:, 4] >= 1).all()
    for lmax in (1, 80):
        rs, qs = eng.exact_knn(Q[0], ssb.QueryConfig(k=5, lmax=lmax))
        od2, oid = oracle.knn_scan(X, Q[:1], 5)
        assert rs.ids() == list(oid[0]) and qs.visited_leaves <= lmax
    del eng, idx  # the graphs are freed with the index
