"""Host overhead of one query call (GPU box): wall time per knn_device call
vs the device time of its kernels (CUDA events around each launch,
ssb_prof_*), for a workload's batch size.

    python tools/call_overhead_probe.py --workload c3 --batch 256 --calls 40
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--calls", type=int, default=40)
    ap.add_argument("--route", default="auto")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2212_13297_b200 import IndexSettings, QueryEngine, _lib, build_index_array

    args = bench.parse(["--workload", a.workload, "--rows", str(a.rows)])
    wl = bench.make_workload(a.workload, args)
    X = torch.from_numpy(wl.data_fn(0, wl.N)).cuda()
    idx = build_index_array(X, IndexSettings(series_length=wl.n, dataset_size=wl.N, leaf_threshold=wl.tau))
    eng = QueryEngine(idx)
    _, fn, k = wl.cells[0]
    Q = torch.from_numpy(fn()[:a.batch]).cuda()
    for _ in range(5):
        eng.knn_device(Q, k, route=a.route)
    torch.cuda.synchronize()
    for prof in (False, True):
        if prof:
            _lib.prof_reset()
            _lib.prof_enable(True)
        walls = []
        for _ in range(a.calls):
            t0 = time.perf_counter()
            eng.knn_device(Q, k, route=a.route)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        if prof:
            _lib.prof_enable(False)
            kern = {name: round(v[0] / a.calls, 4) for name, v in _lib.prof_read().items()}
        walls.sort()
        print(json.dumps({"workload": a.workload, "batch": a.batch, "profiled": prof,
                          "wall_ms_median": round(1000 * walls[len(walls) // 2], 4),
                          "kernel_ms_per_call": kern if prof else None}), flush=True)


if __name__ == "__main__":
    main()
