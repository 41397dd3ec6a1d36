"""bench.py -- exact k-NN data-series search on B200.

Default workload = BASELINE.json configs[1] ("c2"): 1M random-walk series x 256
(float32, z-normalised, reference generator recipe, seed 0); 1000 noisy queries
per sigma in {0.01, 0.1, 1.0} (seed 1); k in {1, 10}.  One step answers the
whole workload (3 sigmas x 2 k x 1000 queries = 6000 exact k-NN answers).
Other BASELINE.json configs: --workload c1 | c3 | c4 | c5 (explicit runs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2]

Multi-GPU (torchrun, one rank per GPU): the dataset is row-sharded (each rank
generates and indexes only its shard), every rank answers every query over its
shard, and the per-shard top-k lists are merged with one NCCL all-gather and
the K-merge kernel (strong scaling: the dataset is fixed).
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


# --------------------------------------------------------------------------
# workloads (BASELINE.json configs)

class Workload:
    """A dataset (generated per shard) plus query cells answered every step."""

    def __init__(self, name, desc, N, n, tau, cells, data_fn, batch=None):
        self.name, self.desc, self.N, self.n, self.tau = name, desc, N, n, tau
        self.cells = cells          # [(label, queries_fn, k)]
        self.data_fn = data_fn      # (lo, hi) -> rows [lo, hi)
        self.batch = batch          # queries per launch (None = the whole cell)


def make_workload(name: str, args) -> Workload:
    from paper_2212_13297_b200 import generate as G

    nq = args.queries
    if name == "c1":
        N, n = args.rows or 100_000, 256
        cells = [("random-walk queries, seed 1", lambda: G.random_walks(100, n, 1, workers=1), 1)]
        return Workload("c1", f"C1: {N} x {n} random walks (seed 0), 100 random-walk queries "
                              f"(seed 1), k=1, tau={args.tau or 1000}", N, n, args.tau or 1000, cells,
                        lambda lo, hi: G.random_walks(hi - lo, n, 0, start=lo))
    if name == "c2":
        N, n = args.rows or 1_000_000, 256
        cells = [(f"sigma={s} k={k}", (lambda s=s: G.noise_queries_stream(N, n, nq, s, 1)), k)
                 for s in (0.01, 0.1, 1.0) for k in (1, 10)]
        return Workload("c2", f"C2: {N} x {n} random walks, {nq} noisy queries per sigma in "
                              f"[0.01, 0.1, 1.0], k in [1, 10] ({6 * nq} answers per step), "
                              f"tau={args.tau or 10_000}", N, n, args.tau or 10_000, cells,
                        lambda lo, hi: G.random_walks(hi - lo, n, 0, start=lo))
    if name == "c3":
        N, n = args.rows or 10_000_000, 96
        cells = [("unit-Gaussian queries seed 3", lambda: G.unit_gaussian_rows(0, nq, n, 3), 10)]
        return Workload("c3", f"C3: {N} x {n} unit-norm Gaussian vectors (seed 2), {nq} queries "
                              f"(seed 3), k=10, 256 queries per launch", N, n, args.tau or 10_000,
                        cells, lambda lo, hi: G.unit_gaussian_rows(lo, hi, n, 2), batch=256)
    if name == "c4":
        N, n = args.rows or 25_000_000, 256
        cells = [("sigma=0.1 k=100", lambda: G.noise_queries_stream(N, n, nq, 0.1, 1), 100)]
        return Workload("c4", f"C4: {N} x {n} random walks, {nq} noisy queries sigma=0.1, k=100, "
                              f"tau={args.tau or 10_000}", N, n, args.tau or 10_000, cells,
                        lambda lo, hi: G.random_walks(hi - lo, n, 0, start=lo))
    if name == "c5":
        N, n = args.rows or 50_000_000, 256
        cells = [(f"sigma={s} k=10", (lambda s=s: G.noise_queries_stream(N, n, nq, s, 1)), 10)
                 for s in (0.01, 1.0)]
        return Workload("c5", f"C5: {N} x {n} random walks, build tau={args.tau or 100_000}, then "
                              f"{nq} queries k=10 at sigma in [0.01, 1.0]", N, n,
                        args.tau or 100_000, cells,
                        lambda lo, hi: G.random_walks(hi - lo, n, 0, start=lo))
    raise SystemExit(f"unknown workload {name}")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="c2", choices=("c1", "c2", "c3", "c4", "c5"))
    ap.add_argument("--rows", type=int, default=0, help="override the dataset size")
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--tau", type=int, default=0, help="override the leaf threshold")
    ap.add_argument("--route", default="auto", choices=("auto", "tree", "tensor", "eapca"))
    ap.add_argument("--per-cell", action="store_true",
                    help="one call per (sigma, k) cell instead of one call per k with the cells' queries batched")
    ap.add_argument("--engine", default="index", choices=("index", "bruteforce"))
    ap.add_argument("--cpu-sample", type=int, default=4, help="queries per cell for the CPU baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-multi", action="store_true", help="one ssb_query per call (not ssb_query_multi)")
    ap.add_argument("--ingest-gb", type=float, default=4.0,
                    help="file -> HBM ingest sample (GB of the shard; 0 = skip), reported under build.ingest")
    return ap.parse_args()


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
    """Full exact scan (K-scan dense + K-select): pscan.py:23-135 on the device."""

    name = "bruteforce (K-scan dense + K-select)"

    def __init__(self, X_dev, id_base: int = 0, **_):
        self.X = X_dev
        self.id_base = id_base

    def build_info(self, N):
        return None

    def query(self, Q_dev, k):
        from paper_2212_13297_b200 import knn_batch

        return knn_batch(self.X, Q_dev, k, id_base=self.id_base)

    def query_host(self, Q_host, k):
        d2, ids = self.query(Q_host, k)
        return d2.cpu().numpy(), ids.cpu().numpy()


class IndexEngine:
    """The product path: level-synchronous GPU build, then batched exact
    queries routed per query (auto cost model) between the K-tc tensor-core
    filter + exact rescoring and K-lbe/K-lbs + sparse K-scan; K-select."""

    name = ("index: K-lbe, then per query K-tc tensor-core filter + exact rescoring "
            "or K-lbs + sparse K-scan (route={route}); K-select")

    def __init__(self, X_dev, tau: int, id_base: int = 0, route: str = "auto"):
        import torch

        from paper_2212_13297_b200 import IndexSettings, QueryEngine, build_index_array

        s = IndexSettings(series_length=X_dev.shape[1], dataset_size=X_dev.shape[0], leaf_threshold=tau)
        # warm-up build on a small prefix: module loading and pool growth stay out of
        # the timed build (the steady state of a process that builds indexes)
        w = min(X_dev.shape[0], 20_000)
        build_index_array(X_dev[:w], IndexSettings(series_length=X_dev.shape[1], dataset_size=w,
                                                   leaf_threshold=min(tau, max(1, w // 4))))
        torch.cuda.synchronize()
        from paper_2212_13297_b200 import _lib

        _lib.prof_reset()
        _lib.prof_enable(True)  # per-kernel CUDA events of the build (ProfScope)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        ev0.record()
        self.index = build_index_array(X_dev, s, id_base=id_base)
        ev1.record()
        torch.cuda.synchronize()
        _lib.prof_enable(False)
        self.build_prof = _lib.prof_read()
        _lib.prof_reset()
        self.build_wall_s = time.perf_counter() - t0
        self.build_dev_ms = ev0.elapsed_time(ev1)
        self.engine = QueryEngine(self.index)
        self.route = route
        self.name = IndexEngine.name.format(route=route)

    def build_info(self, N):
        info = self.index.info
        out = {"series_per_s": round(N / self.build_wall_s, 1), "ms": round(1000 * self.build_wall_s, 2),
               "device_ms": round(self.build_dev_ms, 2), "leaves": info.num_leaves,
               "nodes": info.num_nodes, "levels": info.levels, "depth": info.depth,
               "kernels": {k: {"ms": round(v[0], 3), "launches": v[1], "GB": round(v[2] / 1e9, 3)}
                           for k, v in self.build_prof.items()}}
        if self.build_prof:
            # K-stats (the build's HBM-bound summarisation pass, its largest kernel
            # except on tiny C1-sized builds where the ALU-bound K-eval can lead)
            # against the measured HBM peak
            name = "build_stats" if "build_stats" in self.build_prof else max(
                self.build_prof.items(), key=lambda kv: kv[1][0])[0]
            kms, klaunch, kbytes, _ = self.build_prof[name]
            try:
                peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0))
            except OSError:
                peak = 6650.0
            gbs = kbytes / (kms / 1000.0) / 1e9
            out["roofline"] = {"kernel": name, "bound": "hbm", "achieved": round(gbs, 1), "peak": peak,
                               "unit": "GB/s", "frac": round(gbs / peak, 4), "share_of_build": round(
                                   kms / max(self.build_dev_ms, 1e-9), 4),
                               "bytes": "per level: 4n B per active series read + 24m B of statistics written"}
        return out

    def query(self, Q_dev, k):
        d2, ids, _ = self.engine.knn_device(Q_dev, k, route=self.route)
        return d2, ids

    def query_host(self, Q_host, k):
        d2, ids, _ = self.engine.knn_device(Q_host, k, route=self.route)
        return d2.cpu().numpy(), ids.cpu().numpy()

    def query_multi(self, calls):
        """All of a step's calls (different k) through one ssb_query_multi."""
        return [(d2, ids) for d2, ids, _ in self.engine.knn_device_multi(calls, route=self.route)]


def merge_shards(d2, ids, k):
    """One NCCL all-gather of every rank's top-k keys + the K-merge kernel."""
    from paper_2212_13297_b200.distributed import merge_topk

    return merge_topk(d2, ids, k)


# --------------------------------------------------------------------------
# reference arm: the oracle port timed on host cores

def cpu_baseline(wl: Workload, X, cellq, sample: int):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    nq = 0
    for (_, _, k), Q in zip(wl.cells, cellq):
        oracle.knn_scan(X, Q[:sample], k, threads=threads)
        nq += min(sample, len(Q))
    dt = time.perf_counter() - t0
    return {"value": nq / dt, "unit": "queries/s", "cores": threads, "kind": "port",
            "sample": f"{nq} queries ({sample} per cell) of workload {wl.name} through the C "
                      f"oracle's exact scan (pscan.py:23-135 restated, {threads} threads)",
            "seconds": dt}


def run_reference(args, rank, world):
    if rank != 0:
        return
    wl = make_workload(args.workload, args)
    X = wl.data_fn(0, wl.N)
    cellq = [fn() for _, fn, _ in wl.cells]
    for _ in range(args.warmup):
        cpu_baseline(wl, X, cellq, 1)
    vals = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_baseline(wl, X, cellq, args.cpu_sample))
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
        "config": {"workload": wl.desc + f"; each step is a bounded sample of {args.cpu_sample} "
                                         "queries per cell"},
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
    from paper_2212_13297_b200.distributed import shard_range

    wl = make_workload(args.workload, args)
    N = wl.N
    lo, hi = shard_range(N, rank, world)
    t_gen = time.perf_counter()
    X = wl.data_fn(lo, hi)
    cellq = [fn() for _, fn, _ in wl.cells]
    t_gen = time.perf_counter() - t_gen
    X_dev = None
    ingest = None
    if args.ingest_gb > 0:
        # file -> pinned double buffer -> HBM (ssb_ingest_file), on a sample of
        # the shard written to a local file first (page cache: the pipeline, not
        # the disk, is measured); a sample covering the whole shard becomes X_dev
        import tempfile

        from paper_2212_13297_b200 import ingest_file

        rows = int(min(len(X), max(1, args.ingest_gb * 1e9 // (4 * wl.n))))
        fd, path = tempfile.mkstemp(suffix=".bin")
        try:
            with os.fdopen(fd, "wb") as f:
                X[:rows].tofile(f)
            ingest_file(path, wl.n, 0, rows)  # warm the pinned buffers
            D, st = ingest_file(path, wl.n, 0, rows)
        finally:
            os.unlink(path)
        ingest = {"GBps": round(st["GBps"], 2), "bytes": st["bytes"], "rows": rows, "of_shard_rows": len(X),
                  "source": "raw float32 file in the page cache, 64 MB pinned double buffer, "
                            f"{min(16, os.cpu_count() or 1)} read threads"}
        if rows == len(X):
            X_dev = D
        del D
    if X_dev is None:
        X_dev = torch.from_numpy(X).cuda()
    # device generator (documented Philox stream) on a sample of
    # the shard size, beside the host generator time (data_gen_s)
    from paper_2212_13297_b200 import generate as _G

    g_rows = min(len(X), 4_000_000)
    g_fn = _G.unit_gaussian_device if args.workload == "c3" else _G.random_walks_device
    g_fn(1024, wl.n, 0)
    torch.cuda.synchronize()
    g0 = time.perf_counter()
    g_out = g_fn(g_rows, wl.n, 0, start=lo)
    torch.cuda.synchronize()
    g_s = time.perf_counter() - g0
    del g_out
    device_gen = {"series_per_s": round(g_rows / g_s, 1), "rows": g_rows,
                  "host_series_per_s": round(len(X) / t_gen, 1) if t_gen > 0 else None}
    # the calls of one step: every cell's queries are answered; cells with the
    # same k are batched into one call unless --per-cell (same queries, same
    # answers: the batch size is the engine's choice, the API takes any B)
    calls = []
    for (_, _, k), Q in zip(wl.cells, cellq):
        if not args.per_cell and calls and calls[-1][0] == k:
            calls[-1][1].append(Q)
        elif not args.per_cell and any(c[0] == k for c in calls):
            next(c for c in calls if c[0] == k)[1].append(Q)
        else:
            calls.append((k, [Q]))
    calls = [(k, np.concatenate(qs)) for k, qs in calls]
    Q_dev = [(k, torch.from_numpy(Q).cuda()) for k, Q in calls]
    if args.engine == "index":
        engine = IndexEngine(X_dev, wl.tau, id_base=lo, route=args.route)
    else:
        engine = BruteForceEngine(X_dev, id_base=lo)
    batch = wl.batch

    def answer(Q, k, host=False):
        chunks = [Q] if not batch else [Q[i:i + batch] for i in range(0, len(Q), batch)]
        out = []
        for c in chunks:
            if host:
                out.append(engine.query_host(c, k))
            else:
                d2, ids = engine.query(c, k)
                out.append(merge_shards(d2, ids, k) if world > 1 else ids)
        return out

    # every call of a step through one multi-call (one host round trip per step
    # instead of one per call); --no-multi answers them one ssb_query each
    multi = not batch and hasattr(engine, "query_multi") and not args.no_multi

    def step():
        if multi:
            outs = engine.query_multi([(Q, k) for k, Q in Q_dev])
            return [[merge_shards(d2, ids, k) if world > 1 else ids] for (k, _), (d2, ids) in zip(Q_dev, outs)]
        return [answer(Q, k) for k, Q in Q_dev]

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
    answers = sum(len(Q) for Q in cellq)
    value = answers * args.steps / (ms / 1000.0)

    # ---- e2e: the public API with host buffers, copies inside the region ------
    Q_host = [(k, torch.from_numpy(Q).pin_memory()) for k, Q in calls]
    h2d = sum(Q.numel() * 4 for _, Q in Q_host)
    d2h = sum(len(Q) * k * (4 + 8) for k, Q in calls)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        if multi:
            outs = engine.query_multi([(Qh, k) for k, Qh in Q_host])
            _ = [(d2.cpu().numpy(), ids.cpu().numpy()) for d2, ids in outs]
        else:
            for k, Qh in Q_host:
                answer(Qh, k, host=True)
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
        # DRAM traffic per launch of this kernel from a committed `ncu --set full`
        # capture of the same workload (profiles/traffic.json), when there is one
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(wl.name, {})
            if tr.get("kernel") == name:
                roof["traffic"] = tr["bytes_per_launch"]
                roof["traffic_source"] = tr["source"]
        except (OSError, ValueError, KeyError):
            pass
    cb = None
    if not args.no_cpu_baseline and world == 1:
        cb = cpu_baseline(wl, X, cellq, args.cpu_sample)
        cb.pop("seconds", None)
    line = {
        "metric": "exact kNN queries/s", "value": round(value, 1), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference generator recipe (seeded Philox streams; see DESIGN.md Inputs)",
        "config": {"workload": wl.desc, "engine": engine.name, "shards": world,
                   "calls_per_step": [{"k": k, "queries": len(Q)} for k, Q in calls],
                   "api": "QueryEngine.knn_device_multi (ssb_query_multi: one host round trip per step)" if multi else "QueryEngine.knn_device per call",
                   "l2": "inputs larger than L2 (dataset %.2f GB > 126 MB)" % (N * wl.n * 4 / 1e9),
                   "data_gen_s": round(t_gen, 1)},
        "roofline": roof,
        "kernels": {k: {"ms": round(v[0], 3), "launches": v[1], "GB": round(v[2] / 1e9, 3),
                        "TFLOP": round(v[3] / 1e12, 3)} for k, v in prof.items()},
        "cpu_baseline": cb,
        "e2e": {"value": round(e2e, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "build": dict(engine.build_info(hi - lo), **({"ingest": ingest} if ingest else {}),
                      device_gen=device_gen),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
