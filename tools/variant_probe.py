"""A/B of library switches on one workload, one process, one build (GPU box).

    python tools/variant_probe.py --workload c4 --steps 5 \
        --variants '[{"route": "tensor"}, {"route": "auto", "SSB_SEED_MULT": "8"}]'

Each variant: environment switches (SSB_*; read by the library per call) plus
an optional "route"; prints one JSON line per variant with answers/s over the
timed steps (CUDA events), the per-kernel device times and a parity check of
the first queries against the first variant's answers.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--rows", type=int, default=0)
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--variants", required=True)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2212_13297_b200 import IndexSettings, QueryEngine, _lib, build_index_array

    args = bench.parse(["--workload", a.workload, "--rows", str(a.rows), "--queries", str(a.queries)])
    wl = bench.make_workload(a.workload, args)
    X = torch.from_numpy(wl.data_fn(0, wl.N)).cuda()
    idx = build_index_array(X, IndexSettings(series_length=wl.n, dataset_size=wl.N, leaf_threshold=wl.tau))
    eng = QueryEngine(idx)
    calls = {}
    for (_, fn, k), in [(c,) for c in wl.cells]:
        calls.setdefault(k, []).append(fn())
    calls = [(torch.from_numpy(np.concatenate(v)).cuda(), k) for k, v in calls.items()]
    if wl.batch:  # the workload's queries per launch (C3: 256)
        calls = [(Q[i:i + wl.batch], k) for Q, k in calls for i in range(0, len(Q), wl.batch)]
    ref = None
    for var in json.loads(a.variants):
        var = dict(var)
        route = var.pop("route", "auto")
        old = {k: os.environ.get(k) for k in var}
        os.environ.update({k: str(v) for k, v in var.items()})
        try:
            def step():
                if wl.batch:
                    return [eng.knn_device(Q, k, route=route)[:2] for Q, k in calls]
                return eng.knn_device_multi(calls, route=route)

            for _ in range(2):
                outs = step()
            torch.cuda.synchronize()
            _lib.prof_reset()
            _lib.prof_enable(True)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.steps):
                outs = step()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            _lib.prof_enable(False)
            prof = {k: round(v[0] / a.steps, 3) for k, v in _lib.prof_read().items()}
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        ids = [o[1][:64].cpu().numpy() for o in outs]
        same = None if ref is None else all(np.array_equal(x, y) for x, y in zip(ids, ref))
        ref = ref or ids
        nq = sum(int(c[0].shape[0]) for c in calls)
        print(json.dumps({"variant": dict(var, route=route), "ms_per_step": round(ms, 3),
                          "answers_per_s": round(nq / (ms / 1000), 1), "kernels_ms": prof,
                          "same_ids_as_first": same}), flush=True)


if __name__ == "__main__":
    main()
