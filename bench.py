"""bench.py -- exact k-NN data-series search on B200.

Default workload = BASELINE.json configs[1] ("C2"): 1M random-walk series x 256
(float32, z-normalised, reference generator recipe, seed 0); 1000 noisy queries
per sigma in {0.01, 0.1, 1.0} (seed 1); k in {1, 10}.  One step answers the
whole workload (3 sigmas x 2 k x 1000 queries = 6000 exact k-NN answers).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): the dataset is row-sharded, every rank
answers every query over its shard, and per-shard top-k lists are merged with
one NCCL all-gather (strong scaling: the dataset is fixed).
Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIGMAS = (0.01, 0.1, 1.0)
KS = (1, 10)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--tau", type=int, default=10_000)
    ap.add_argument("--engine", default="index", choices=("index", "bruteforce"))
    ap.add_argument("--cpu-sample", type=int, default=4, help="queries per (sigma,k) cell "
                    "for the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------------------
# data (reference generator recipe)

def make_inputs(rows: int, n: int, queries: int):
    from paper_2212_13297_b200 import generate as G

    X = G.random_walks(rows, n, 0)
    Qs = {s: G.noise_queries(X, queries, s, 1) for s in SIGMAS}
    return X, Qs


# --------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------
# engines

class BruteForceEngine:
    """Full exact scan (K-scan dense + K-select) -- the reference's own
    exactness path (pscan.py:23-30 / 33-135) on the device."""

    name = "bruteforce (K-scan dense + K-select)"

    def __init__(self, X_dev, id_base: int = 0):
        self.X = X_dev
        self.id_base = id_base

    def query(self, Q_dev, k):
        from paper_2212_13297_b200 import knn_batch

        return knn_batch(self.X, Q_dev, k, id_base=self.id_base)


class IndexEngine:
    """The product path: level-synchronous GPU build, then batched pruned
    exact queries (K-lbe -> K-lbs -> sparse K-scan -> K-select)."""

    name = ("index: K-lbe seed/route, then per query K-tc tensor-core filter + exact rescoring "
            "or K-lbs + sparse K-scan (auto cost model); K-select")

    def __init__(self, X_dev, tau: int, id_base: int = 0):
        import torch

        from paper_2212_13297_b200 import IndexSettings, QueryEngine, build_index_array

        s = IndexSettings(series_length=X_dev.shape[1], dataset_size=X_dev.shape[0], leaf_threshold=tau)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        self.index = build_index_array(X_dev, s, id_base=id_base)
        ev1.record()
        torch.cuda.synchronize()
        self.build_wall_s = time.perf_counter() - t0
        self.build_dev_ms = ev0.elapsed_time(ev1)
        self.engine = QueryEngine(self.index)
        self.id_base = id_base

    def build_info(self, N):
        info = self.index.info
        return {"series_per_s": round(N / self.build_wall_s, 1), "ms": round(1000 * self.build_wall_s, 2),
                "device_ms": round(self.build_dev_ms, 2), "leaves": info.num_leaves,
                "nodes": info.num_nodes, "levels": info.levels, "depth": info.depth}

    def query(self, Q_dev, k):
        d2, ids, _ = self.engine.knn_device(Q_dev, k)
        return d2, ids

    def query_host(self, Q_host, k):
        return self.engine.exact_knn_arrays(Q_host, k)


def merge_shards(d2, ids, k, world):
    """One NCCL all-gather of every rank's top-k keys + the K-merge kernel."""
    from paper_2212_13297_b200.distributed import merge_topk

    return merge_topk(d2, ids, k)


# --------------------------------------------------------------------------
# reference arm: the oracle port timed on host cores

def cpu_baseline(X, Qs, sample: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    nq = 0
    for s in SIGMAS:
        for k in KS:
            oracle.knn_scan(X, Qs[s][:sample], k, threads=threads)
            nq += sample
    dt = time.perf_counter() - t0
    return {"value": nq / dt, "unit": "queries/s", "cores": threads, "kind": "port",
            "sample": f"{nq} queries ({sample} per sigma x k cell) of the C2 workload through the "
                      f"C oracle's exact scan (pscan.py:23-135 restated, {threads} threads)",
            "seconds": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return
    X, Qs = make_inputs(args.rows, args.n, args.queries)
    for _ in range(args.warmup):
        cpu_baseline(X, Qs, 1)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(X, Qs, args.cpu_sample))
    total = time.perf_counter() - t0
    nq = sum(v["value"] * v["seconds"] for v in vals)
    value = nq / sum(v["seconds"] for v in vals)
    cb = dict(vals[-1])
    cb["value"] = value
    cb.pop("seconds", None)
    line = {
        "impl": "reference", "metric": "exact kNN queries/s", "value": value, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator recipe)",
        "config": {"workload": f"C2: {args.rows} x {args.n} random walks, {args.queries} queries per "
                               f"sigma in {list(SIGMAS)}, k in {list(KS)}; each step is a bounded "
                               f"sample of {args.cpu_sample} queries per cell"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------

def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2212_13297_b200 import _lib

    X, Qs = make_inputs(args.rows, args.n, args.queries)
    N = X.shape[0]
    lo = rank * N // world
    hi = (rank + 1) * N // world
    X_dev = torch.from_numpy(X[lo:hi]).cuda()
    Q_dev = {s: torch.from_numpy(Qs[s]).cuda() for s in SIGMAS}
    if args.engine == "index":
        engine = IndexEngine(X_dev, args.tau, id_base=lo)
    else:
        engine = BruteForceEngine(X_dev, id_base=lo)

    def step():
        outs = []
        for s in SIGMAS:
            for k in KS:
                d2, ids = engine.query(Q_dev[s], k)
                if world > 1:
                    outs.append(merge_shards(d2, ids, k, world))
                else:
                    outs.append(ids)
        return outs

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device-timed, max over ranks) -------------------------
    _lib.prof_reset()
    _lib.prof_enable(True)
    launches0 = _lib.launch_count()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = _lib.launch_count() - launches0
    _lib.prof_enable(False)
    prof = _lib.prof_read()
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    answers = len(SIGMAS) * len(KS) * args.queries
    value = answers * args.steps / (ms / 1000.0)

    # ---- e2e: the public API with host buffers, copies inside the region ------
    from paper_2212_13297_b200 import knn_batch

    Q_host = {s: torch.from_numpy(Qs[s]).pin_memory() for s in SIGMAS}
    if args.engine == "index":
        def host_call(Qh, k):
            return engine.query_host(Qh, k)
    else:
        def host_call(Qh, k):
            d2, ids = knn_batch(X_dev, Qh, k, id_base=lo)
            return d2.cpu(), ids.cpu()
    h2d = sum(Q_host[s].numel() * 4 for s in SIGMAS) * len(KS)
    d2h = sum(args.queries * k * (4 + 8) for k in KS) * len(SIGMAS)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for s in SIGMAS:
            for k in KS:
                host_call(Q_host[s], k)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = answers * args.steps / e2e_s

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # ---- roofline of the dominant kernel ---------------------------------------
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    top = max(prof.items(), key=lambda kv: kv[1][0]) if prof else None
    roof = None
    if top:
        name, (kms, klaunch, kbytes, kflops) = top
        avg_s = (kms / klaunch) / 1000.0
        if kflops > 0:  # tensor-core kernel: FLOPs against the measured bf16 peak
            tf_peak = float(peaks.get("bf16_tflops", 1590.0))
            achieved = (kflops / klaunch) / avg_s / 1e12
            roof = {"kernel": name, "bound": "tensor", "achieved": round(achieved, 1), "peak": tf_peak,
                    "unit": "TFLOP/s", "frac": round(achieved / tf_peak, 4), "traffic": None,
                    "hbm_GBps": round((kbytes / klaunch) / avg_s / 1e9, 1),
                    "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if peaks else "fallback 1.59 PF"}
        else:
            achieved = (kbytes / klaunch) / avg_s / 1e9
            roof = {"kernel": name, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
        roof.update({"share_of_step": round(kms / ms, 4), "avg_launch_ms": round(kms / klaunch, 4)})
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(X, Qs, args.cpu_sample)
        cb.pop("seconds", None)
    line = {
        "metric": "exact kNN queries/s", "value": round(value, 1), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference generator recipe (Philox random walks, seed 0; noisy queries, seed 1)",
        "config": {"workload": f"C2: {N} x {args.n} random walks, {args.queries} queries per sigma in "
                               f"{list(SIGMAS)}, k in {list(KS)} ({answers} answers per step)",
                   "engine": engine.name, "shards": world,
                   "l2": "inputs larger than L2 (dataset %.2f GB > 126 MB)" % (X.nbytes / 1e9)},
        "roofline": roof,
        "kernels": {k: {"ms": round(v[0], 3), "launches": v[1], "GB": round(v[2] / 1e9, 3),
                        "TFLOP": round(v[3] / 1e12, 3)} for k, v in prof.items()},
        "cpu_baseline": cb,
        "e2e": {"value": round(e2e, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "build": engine.build_info(N) if args.engine == "index" else None,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
