"""Single-query exact k-NN on the GPU box: latency of one query per call on
each path over N device-resident rows (the device generator's random walks:
no host generation), for ncu captures of the single-query kernels.

    python tools/single_scan_probe.py --rows 25000000 --k 100 --calls 20

Paths: "scan" = ssb_bruteforce_knn (pscan.brute_force_knn; for B <= 4 the
row-parallel early-abandoning scan_rows_kernel), "tensor" / "tree" / "auto" =
QueryEngine.knn_device through the index (the tensor route streams the BF16
operand once for a 1-query block).
"""
import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=25_000_000)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--calls", type=int, default=20)
    ap.add_argument("--paths", default="scan,tensor,tree,auto")
    a = ap.parse_args()
    import torch

    from paper_2212_13297_b200 import IndexSettings, QueryEngine, build_index_array, generate, knn_batch

    X = generate.random_walks_device(a.rows, a.n, 0)
    Qs = generate.random_walks_device(a.calls + 2, a.n, 1)
    eng = None
    for path in a.paths.split(","):
        if path != "scan" and eng is None:
            idx = build_index_array(X, IndexSettings(series_length=a.n, dataset_size=a.rows, leaf_threshold=10_000))
            eng = QueryEngine(idx)
        lat = []
        for i in range(a.calls + 2):
            q = Qs[i:i + 1]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if path == "scan":
                d2, ids = knn_batch(X, q, a.k)
            else:
                d2, ids, _ = eng.knn_device(q, a.k, route=path)
            torch.cuda.synchronize()
            if i >= 2:
                lat.append(time.perf_counter() - t0)
        print(json.dumps({"path": path, "rows": a.rows, "n": a.n, "k": a.k, "median_ms": round(1000 * statistics.median(lat), 4),
                          "p90_ms": round(1000 * sorted(lat)[int(0.9 * len(lat))], 4),
                          "row_GBps_at_median": round(a.rows * a.n * 4 / statistics.median(lat) / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
