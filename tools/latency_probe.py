"""Single-query latency and per-cell routes on the GPU box.

    python tools/latency_probe.py --workload c2 [--rows N] [--queries 50]

For each cell of the workload: the median latency of ONE query per call
(QueryEngine.exact_knn, the reference's own per-query API, host buffers) on
each route, the rows the index route reads, and batched answers/s of the whole
cell per route; every answer is checked against the oracle (test
infrastructure, as the checker).  Prints one JSON line per (cell, route).
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--single", type=int, default=30, help="single-query calls timed per route")
    ap.add_argument("--routes", default="tree,tensor,auto")
    ap.add_argument("--check", type=int, default=8, help="answers per cell checked against the oracle")
    a = ap.parse_args()
    import torch

    import bench
    import oracle
    from paper_2212_13297_b200 import IndexSettings, QueryConfig, QueryEngine, _lib, build_index_array

    args = bench.parse(["--workload", a.workload, "--rows", str(a.rows), "--queries", str(a.queries)])
    wl = bench.make_workload(a.workload, args)
    X = wl.data_fn(0, wl.N)
    Xd = torch.from_numpy(X).cuda()
    idx = build_index_array(Xd, IndexSettings(series_length=wl.n, dataset_size=wl.N, leaf_threshold=wl.tau))
    eng = QueryEngine(idx)
    routes = a.routes.split(",")
    import paper_2212_13297_b200 as ssb

    for label, fn, k in wl.cells[:1]:
        # the brute-force scan of ONE query (pscan.brute_force_knn; B <= 4 takes
        # the row-parallel early-abandoning scan): latency and scan-equivalent GB/s
        Q = fn()
        od2, oid = oracle.knn_scan(X, Q[:3], k, threads=os.cpu_count())
        lat, ok = [], True
        _lib.prof_reset()
        _lib.prof_enable(True)
        for i in range(a.single + 2):
            q = torch.from_numpy(Q[i % 3:i % 3 + 1]).cuda()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d2, ids = ssb.knn_batch(Xd, q, k)
            torch.cuda.synchronize()
            if i >= 2:
                lat.append(time.perf_counter() - t0)
            ok &= bool(np.array_equal(ids.cpu().numpy()[0], oid[i % 3]))
        _lib.prof_enable(False)
        kp = _lib.prof_read()
        ms = statistics.median(lat) * 1000
        print(json.dumps({"workload": wl.name, "cell": label, "k": k, "route": "bruteforce B=1",
                          "single_ms_median": round(ms, 3), "parity_ok": ok,
                          "scan_equivalent_GBps": round(wl.N * wl.n * 4 / (ms / 1000) / 1e9, 1),
                          "kernels_ms_GB": {kk: [round(v[0] / (a.single + 2), 4), round(v[2] / (a.single + 2) / 1e9, 3)]
                                            for kk, v in kp.items()}}), flush=True)
    for label, fn, k in wl.cells:
        Q = fn()
        od2, oid = oracle.knn_scan(X, Q[:a.check], k, threads=os.cpu_count())
        for route in routes:
            # batched: the whole cell in one call
            Qd = torch.from_numpy(Q).cuda()
            eng.knn_device(Qd, k, route=route)
            torch.cuda.synchronize()
            _lib.prof_reset()
            _lib.prof_enable(True)
            t0 = time.perf_counter()
            reps = 3
            for _ in range(reps):
                d2, ids, _ = eng.knn_device(Qd, k, route=route)
            torch.cuda.synchronize()
            batch_qps = reps * len(Q) / (time.perf_counter() - t0)
            _lib.prof_enable(False)
            bprof = {kk: [round(v[0] / reps, 3), v[1] // reps, round(v[2] / reps / 1e9, 4)]
                     for kk, v in _lib.prof_read().items()}
            ok = np.array_equal(ids[:a.check].cpu().numpy(), oid) and np.array_equal(
                d2[:a.check].cpu().numpy().view(np.uint32), od2.view(np.uint32))
            # single queries through the device API, then the host API (exact_knn)
            lat, lat_host, stats = [], [], []
            _lib.prof_reset()
            _lib.prof_enable(True)
            for i in range(a.single + 2):
                q = Qd[i % len(Q):i % len(Q) + 1]
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                d2s, ids1, _, st = eng.knn_device(q, k, route=route, want_stats=True)
                torch.cuda.synchronize()
                if i >= 2:
                    lat.append(time.perf_counter() - t0)
                    stats.append(st[0])
            _lib.prof_enable(False)
            sprof = {kk: [round(v[0] / (a.single + 2), 4), round(v[2] / (a.single + 2) / 1e6, 3)]
                     for kk, v in _lib.prof_read().items()}
            cfg = QueryConfig(k=k)
            for i in range(a.single + 2):
                t0 = time.perf_counter()
                rs, qs = eng.exact_knn(Q[i % len(Q)], cfg) if route == "auto" else (None, None)
                if route != "auto":
                    break
                if i >= 2:
                    lat_host.append(time.perf_counter() - t0)
            st = np.array(stats, dtype=np.float64)
            print(json.dumps({
                "workload": wl.name, "cell": label, "k": k, "route": route, "batch_queries": len(Q),
                "batch_answers_per_s": round(batch_qps, 1), "parity_ok": bool(ok),
                "single_ms_median": round(1000 * statistics.median(lat), 3),
                "batch_kernels_ms_launches_GB": bprof, "single_kernels_ms_MB": sprof,
                "exact_knn_ms_median": round(1000 * statistics.median(lat_host), 3) if lat_host else None,
                "single_stats_mean": {"cand_leaves": st[:, 0].mean(), "cand_series": st[:, 1].mean(),
                                      "seed_rows": st[:, 2].mean(), "seed_leaves": st[:, 4].mean(),
                                      "words": st[:, 5].mean(), "abandoned": st[:, 6].mean(),
                                      "tc": st[:, 7].mean()}}), flush=True)


if __name__ == "__main__":
    main()
