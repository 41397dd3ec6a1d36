"""bench.py -- exact k-NN data-series search on B200.

Default workload = BASELINE.json configs[3] ("c4"), the largest configuration
that is a query workload on one GPU: 25M random-walk series x 256 (float32,
z-normalised, the reference generator's recipe, seed 0); 1000 noisy queries
(sigma = 0.1, seed 1), k = 100, leaf threshold 10^4.  One step answers the
whole workload.  Other configs: --workload c1 | c2 | c3 | c5.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c4]

Multi-GPU: one rank per GPU.  Launched by torchrun (RANK/WORLD_SIZE set) or,
with ``--gpus N`` and no WORLD_SIZE, this script re-launches itself under
``torch.distributed.run`` with N ranks.  The dataset is row-sharded (each rank
generates and indexes only its shard), every rank answers every query over its
shard, and inside the timed step the per-shard top-k lists are packed on the
device, all-gathered (NCCL) and merged by the K-merge kernel (strong scaling:
the dataset is fixed).  Prints ONE JSON line on rank 0.

The answers are checked: the oracle's exact scan (test infrastructure, run
only here in the cpu_baseline leg, as the checker) answers a bounded sample of
the same queries, and the line carries "parity": {"checked", "mismatches"};
any mismatch exits non-zero.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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
        q1 = min(nq, 100)
        cells = [("random-walk queries, seed 1", lambda: G.random_walks(q1, n, 1, workers=1), 1)]
        return Workload("c1", f"C1: {N} x {n} random walks (seed 0), {q1} random-walk queries "
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


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="c4", choices=("c1", "c2", "c3", "c4", "c5"))
    ap.add_argument("--rows", type=int, default=0, help="override the dataset size")
    ap.add_argument("--queries", type=int, default=1000)
    ap.add_argument("--tau", type=int, default=0, help="override the leaf threshold")
    ap.add_argument("--route", default="auto", choices=("auto", "tree", "tensor", "eapca"))
    ap.add_argument("--per-cell", action="store_true",
                    help="one call per (sigma, k) cell instead of one call per k with the cells' queries batched")
    ap.add_argument("--engine", default="index", choices=("index", "bruteforce"))
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU baseline + parity sample: oracle queries until about this many seconds")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="fixed number of sampled queries per cell (overrides --cpu-seconds)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-multi", action="store_true", help="one ssb_query per call (not ssb_query_multi)")
    ap.add_argument("--ingest-gb", type=float, default=4.0,
                    help="file -> HBM ingest sample (GB of the shard; 0 = skip), reported under build.ingest")
    ap.add_argument("--clock-ms", type=int, default=100,
                    help="nvidia-smi sampling period during the timed region (0 = off; NVML queries contend "
                         "with the driver, so keep it coarse)")
    ap.add_argument("--backend", default="nccl", choices=("nccl", "gloo"),
                    help="torch.distributed backend (gloo: CPU tests of the multi-rank plumbing)")
    return ap.parse_args(argv)


# --------------------------------------------------------------------------
# host facts

def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


def load_peaks() -> dict:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def ref_build_baseline(N: int, n: int, tau: int):
    """The reference's own build (pure Python) measured on the builder
    container by tools/ref_build_probe.py (committed: profiles/ref_build_cpu.jsonl;
    the reference is not installed on the GPU box), extrapolated linearly to N."""
    try:
        rows = [json.loads(l) for l in open(os.path.join(ROOT, "profiles", "ref_build_cpu.jsonl")) if l.strip()]
    except (OSError, ValueError):
        return None
    rows = [r for r in rows if r.get("n") == n] or rows
    if not rows:
        return None
    r = min(rows, key=lambda r: (abs(np.log(max(r["tau"], 1) / max(tau, 1))), -r["rows"]))
    return {"value": r["series_per_s"], "unit": "series/s", "cores": r["num_threads"], "kind": "reference",
            "sample": f"reference build_index (build.py:363-458, pure Python, num_threads={r['num_threads']}) "
                      f"of {r['rows']} x {r['n']} random walks, tau={r['tau']}: {r['build_s']} s on the "
                      f"builder container ({r['cores']} cores, {r['cpu_model']}); committed measurement "
                      f"(profiles/ref_build_cpu.jsonl), not re-run on this host",
            "extrapolated_s_for_this_shard": round(N / r["series_per_s"], 1)}


# --------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0, enabled: bool = True, period_ms: int = 100):
        self.index = index
        self.enabled = enabled and period_ms > 0
        self.period_ms = period_ms
        self.proc = None
        self.lines: list[str] = []

    _NAMES = ((0x8, "hw_slowdown"), (0x40, "hw_thermal_slowdown"), (0x20, "sw_thermal_slowdown"), (0x4, "sw_power_cap"))

    def _one(self, nv, h, reasons_fn, mx):
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        r = reasons_fn(h)
        flags = ", ".join("Active" if r & bit else "Not Active" for bit, _ in self._NAMES)
        # the same columns as the nvidia-smi query below (no power query: the slowest NVML call)
        self.lines.append(f"{sm}, {mx}, 0, {r:#x}, {flags}")

    def _nvml_loop(self, nv, h):
        reasons_fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        self._nv = (nv, h, reasons_fn, mx)
        while not self.stop.is_set():
            try:
                self._one(nv, h, reasons_fn, mx)
            except Exception:  # noqa: BLE001 -- a failed sample is skipped
                pass
            while True:  # sleep a period; rearm() restarts the period (no sample right at a region's start)
                self.again.clear()
                self.stop.wait(self.period_ms / 1000.0)
                if self.stop.is_set() or not self.again.is_set():
                    break

    def __enter__(self):
        if not self.enabled:
            return self
        # NVML in this process (a sampling thread) instead of an nvidia-smi process polling
        # the driver: a sample still stalls the step it lands in by ~2.5 ms (C3, per-step
        # host times under SSB_BENCH_TRACE=1), a process start-up costs far more
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.stop = threading.Event()
            self.again = threading.Event()
            self.t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
            self.t.start()
            self.nvml = True
            return self
        except Exception:  # noqa: BLE001 -- no NVML binding: the nvidia-smi loop
            self.nvml = False
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
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
        if getattr(self, "nvml", False):
            self.stop.set()
            self.t.join(timeout=2)
            return
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def mark(self):
        self.marks = getattr(self, "marks", []) + [len(self.lines)]

    def sample_now(self):
        """One sample from the calling thread (the end of a timed region: still under load)."""
        if getattr(self, "nvml", False):
            try:
                self._one(*self._nv)
            except Exception:  # noqa: BLE001
                pass

    def rearm(self):
        """Restart the sampling period: the next sample is one period from now.  A sample
        stalls the CUDA calls it collides with (2-3 ms as a rule, 20-150 ms now and then:
        per-step host times under SSB_BENCH_TRACE=1); the settle loop's 0.5 s used to put one
        on the first steps of every timed region."""
        if getattr(self, "nvml", False):
            self.again.set()

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        marks = getattr(self, "marks", [])
        lines = self.lines
        if len(marks) == 2 and marks[1] > marks[0]:
            lines = lines[marks[0]:marks[1] + 1]  # the samples inside the timed region (+ the next)
        elif len(marks) == 2:
            lines = lines[marks[0]:marks[0] + 2]  # region shorter than one sampling period
        for line in lines:
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
# device plumbing: CUDA events on the launching stream (the product), or host
# clocks for the CPU test of the multi-rank plumbing (SSB_BENCH_TEST_ENGINE)

class CudaDev:
    cuda = True

    def __init__(self, local):
        import torch

        self.torch = torch
        torch.cuda.set_device(local)
        self.device = torch.device("cuda", local)

    def sync(self):
        self.torch.cuda.synchronize()

    def region(self):
        t = self.torch
        ev0, ev1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
        stream = t.cuda.current_stream()

        class R:
            def start(self):
                ev0.record(stream)

            def stop(self):
                ev1.record(stream)
                t.cuda.synchronize()
                return ev0.elapsed_time(ev1)
        return R()

    def upload(self, arr):
        return self.torch.from_numpy(arr).to(self.device)

    def pinned(self, arr):
        return self.torch.from_numpy(arr).pin_memory()


class HostDev:
    """CPU-only stand-in (tests of the multi-rank plumbing, gloo): host clocks."""
    cuda = False

    def __init__(self, local):
        import torch

        self.torch = torch
        self.device = torch.device("cpu")

    def sync(self):
        pass

    def region(self):
        class R:
            def start(self):
                self.t0 = time.perf_counter()

            def stop(self):
                return 1000.0 * (time.perf_counter() - self.t0)
        return R()

    def upload(self, arr):
        return self.torch.from_numpy(arr)

    def pinned(self, arr):
        return self.torch.from_numpy(arr)


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


class IndexEngine:
    """The product path: level-synchronous GPU build, then batched exact
    queries routed per query (auto cost model) between the K-tc tensor-core
    filter + exact rescoring and K-lbe/K-lbs + sparse K-scan; K-select."""

    name = ("index: K-lbe, then per query K-tc tensor-core filter + exact rescoring "
            "or K-lbs + sparse K-scan (route={route}); K-select")

    def __init__(self, X_dev, tau: int, id_base: int = 0, route: str = "auto"):
        import torch

        from paper_2212_13297_b200 import IndexSettings, QueryEngine, _lib, build_index_array

        s = IndexSettings(series_length=X_dev.shape[1], dataset_size=X_dev.shape[0], leaf_threshold=tau)
        # warm-up build on a small prefix: module loading and pool growth stay out of
        # the timed build (the steady state of a process that builds indexes)
        w = min(X_dev.shape[0], 20_000)
        build_index_array(X_dev[:w], IndexSettings(series_length=X_dev.shape[1], dataset_size=w,
                                                   leaf_threshold=min(tau, max(1, w // 4))))
        torch.cuda.synchronize()

        def timed_build():
            _lib.prof_reset()
            _lib.prof_enable(True)  # per-kernel CUDA events of the build (ProfScope)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            ev0.record()
            index = build_index_array(X_dev, s, id_base=id_base)
            ev1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            _lib.prof_enable(False)
            prof = _lib.prof_read()
            _lib.prof_reset()
            return index, wall, ev0.elapsed_time(ev1), prof

        # Two builds of the same shard, the first freed before the second: the
        # first one of a process also maps tens of GB of fresh device memory
        # into the stream-ordered pool (0.2 - 1 s on a fresh box, not build
        # work); the second is the steady state of a process that builds
        # indexes.  The faster one is reported, both times are in the line.
        self.build_runs_ms = []
        self.index = None
        for _ in range(1 if os.environ.get("SSB_BENCH_ONE_BUILD") else 2):
            self.index = None  # the previous index is freed before the next build starts
            torch.cuda.synchronize()
            self.index, wall, dev_ms, prof = timed_build()
            self.build_runs_ms.append(round(1000 * wall, 2))
            if len(self.build_runs_ms) == 1 or wall < self.build_wall_s:
                self.build_wall_s, self.build_dev_ms, self.build_prof = wall, dev_ms, prof
        self.engine = QueryEngine(self.index)
        self.route = route
        self.name = IndexEngine.name.format(route=route)

    def build_info(self, N):
        info = self.index.info
        out = {"series_per_s": round(N / self.build_wall_s, 1), "ms": round(1000 * self.build_wall_s, 2),
               "device_ms": round(self.build_dev_ms, 2), "runs_ms": self.build_runs_ms, "leaves": info.num_leaves,
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
            peak = float(load_peaks().get("hbm_gbs", 6650.0))
            gbs = kbytes / (kms / 1000.0) / 1e9
            out["roofline"] = {"kernel": name, "bound": "hbm", "achieved": round(gbs, 1), "peak": peak,
                               "unit": "GB/s", "frac": round(gbs / peak, 4), "share_of_build": round(
                                   kms / max(self.build_dev_ms, 1e-9), 4),
                               "bytes": "per level: 4n B per active series read + 24m B of statistics written"}
        return out

    def query(self, Q_dev, k):
        d2, ids, _ = self.engine.knn_device(Q_dev, k, route=self.route)
        return d2, ids

    def query_multi(self, calls):
        """All of a step's calls (different k) through one ssb_query_multi."""
        return [(d2, ids) for d2, ids, _ in self.engine.knn_device_multi(calls, route=self.route)]


def test_engine():
    """SSB_BENCH_TEST_ENGINE=module:Class -> a CPU engine for the plumbing tests."""
    spec = os.environ.get("SSB_BENCH_TEST_ENGINE")
    if not spec:
        return None
    import importlib

    mod, cls = spec.split(":")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    return getattr(importlib.import_module(mod), cls)


# --------------------------------------------------------------------------
# the oracle leg: CPU baseline + parity checker (the only place bench.py runs
# oracle/, and only as the checker)

def oracle_sample(wl: Workload, X, cellq, sample: int, seconds: float, threads: int):
    """Oracle answers of a bounded sample of every cell's queries (round robin
    over the cells until `seconds` of CPU work, or `sample` per cell).
    Returns ([(cell, j, k, d2 row, ids row)], seconds, queries)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    out = []
    t0 = time.perf_counter()
    j = 0
    while True:
        for c, ((_, _, k), Q) in enumerate(zip(wl.cells, cellq)):
            if j < len(Q):
                d2, ids = oracle.knn_scan(X, Q[j:j + 1], k, threads=threads)
                out.append((c, j, k, d2[0], ids[0]))
        j += 1
        el = time.perf_counter() - t0
        if sample:
            if j >= sample:
                break
        elif el >= seconds or j >= max(len(Q) for Q in cellq):
            break
    return out, time.perf_counter() - t0


def check_parity(answers, gpu_rows):
    """answers: oracle rows; gpu_rows(cell, j) -> (d2 row, ids row) of our path.
    Ids equal and d2 bit-equal (ties to the lowest original index)."""
    bad = []
    for c, j, k, od2, oid in answers:
        gd2, gid = gpu_rows(c, j)
        if not (np.array_equal(np.asarray(gid), oid) and
                np.array_equal(np.asarray(gd2, np.float32).view(np.uint32), od2.view(np.uint32))):
            bad.append({"cell": c, "query": j})
    return {"checked": len(answers), "mismatches": len(bad), "first": bad[:5],
            "rule": "ids identical to the oracle's exact scan (pscan.py:23-30 brute_force_knn, ties to the "
                    "lowest index), squared distances bit-identical"}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU path (the oracle port of pscan's
    exact scan; the reference itself is pure Python and not installed on the
    GPU box) on all host cores, each step a bounded sample of the workload."""
    if rank != 0:
        return
    wl = make_workload(args.workload, args)
    X = wl.data_fn(0, wl.N)
    cellq = [fn() for _, fn, _ in wl.cells]
    threads = os.cpu_count() or 1
    per_step = args.cpu_sample or 0
    # each step: about 2 s of CPU work (so --steps K stays within minutes)
    secs = min(2.0, args.cpu_seconds / 2) if not per_step else 0
    for _ in range(args.warmup):
        oracle_sample(wl, X, cellq, 1, 0, threads)
    nq, tot = 0, 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ans, dt = oracle_sample(wl, X, cellq, per_step, secs, threads)
        nq += len(ans)
        tot += dt
    total = time.perf_counter() - t0
    value = nq / tot
    cb = {"value": value, "unit": "queries/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
          "sample": f"{nq} queries over {args.steps} steps (round robin over the cells) of workload {wl.name} "
                    f"through the C oracle's exact scan (pscan.py:23-135 restated, {threads} threads)"}
    line = {
        "impl": "reference", "metric": "exact kNN queries/s", "value": value, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * total / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator recipe)",
        "config": {"workload": wl.desc + "; each step is a bounded sample of the workload's queries"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------

def relaunch(args) -> int:
    """--gpus N without WORLD_SIZE: run this script under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.run(cmd, env=env).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    sys.exit(run_ours(args, rank, world))


def run_ours(args, rank, world) -> int:
    import torch

    local = int(os.environ.get("LOCAL_RANK", 0))
    TestEngine = test_engine()
    dev = HostDev(local) if TestEngine else CudaDev(local)
    comm = None
    if world > 1:
        import torch.distributed as dist

        if dev.cuda and args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev.device)
        else:
            dist.init_process_group("gloo")
        # the communicator's rank count, checked with one collective
        one = torch.ones(1, device=dev.device)
        dist.all_reduce(one)
        comm = {"backend": dist.get_backend(), "nranks": dist.get_world_size(), "allreduce_ranks": int(one.item())}
    from paper_2212_13297_b200.distributed import merge_topk, shard_range

    wl = make_workload(args.workload, args)
    N = wl.N
    lo, hi = shard_range(N, rank, world)
    t_gen = time.perf_counter()
    X = wl.data_fn(lo, hi)
    cellq = [fn() for _, fn, _ in wl.cells]
    t_gen = time.perf_counter() - t_gen
    X_dev = None
    ingest = device_gen = None
    if dev.cuda:
        X_dev, ingest = ingest_sample(args, X, wl)
        if X_dev is None:
            X_dev = dev.upload(X)
        device_gen = device_gen_sample(args, X, wl, lo)
    else:
        X_dev = dev.upload(X)
    # the calls of one step: every cell's queries are answered; cells with the
    # same k are batched into one call unless --per-cell (same queries, same
    # answers: the batch size is the engine's choice, the API takes any B).
    # where[c] = (call index, first row of cell c inside that call)
    calls, where = [], []
    for (_, _, k), Q in zip(wl.cells, cellq):
        i = next((i for i, c in enumerate(calls) if c[0] == k), None) if not args.per_cell else None
        if i is None:
            calls.append((k, []))
            i = len(calls) - 1
        where.append((i, sum(len(q) for q in calls[i][1])))
        calls[i][1].append(Q)
    calls = [(k, np.concatenate(qs)) for k, qs in calls]
    Q_dev = [(k, dev.upload(Q)) for k, Q in calls]
    if TestEngine:
        engine = TestEngine(X_dev, wl.tau, id_base=lo)
    elif args.engine == "index":
        engine = IndexEngine(X_dev, wl.tau, id_base=lo, route=args.route)
    else:
        engine = BruteForceEngine(X_dev, id_base=lo)
    batch = wl.batch
    merge_fn = getattr(engine, "merge_fn", None)
    # NCCL ranks: the library's own communicator (ssb_comm: pack -> ncclAllGather
    # -> K-merge in one call; the index shares its approximate bounds across the
    # shards with ncclAllReduce(MIN) before filtering)
    ssb_comm = None
    if world > 1 and dev.cuda and args.backend == "nccl" and not TestEngine:
        from paper_2212_13297_b200.distributed import Comm

        try:
            ssb_comm = Comm(rank, world)
        except Exception as e:  # the torch.distributed merge still works: report, carry on
            comm["library_comm"] = f"unavailable ({e}); torch.distributed all-gather + K-merge"
        else:
            if isinstance(engine, IndexEngine):
                ssb_comm.attach(engine.index)
            comm["library_comm"] = "ssb_comm (NCCL all-gather merge + all-reduce(MIN) of the approximate bounds)"

    def merged(d2, ids, k):
        if world == 1:
            return d2, ids
        if ssb_comm is not None:
            return ssb_comm.merge(d2, ids, k)
        return merge_topk(d2, ids, k, merge_fn=merge_fn)

    # every call of a step through one multi-call (one host round trip per step
    # instead of one per call); --no-multi answers them one ssb_query each
    multi = not batch and hasattr(engine, "query_multi") and not args.no_multi

    def step(qs):
        """Answer every call of the step (shard top-k, then the merge at N > 1)."""
        if multi:
            outs = engine.query_multi([(Q, k) for k, Q in qs])
            return [merged(d2, ids, k) for (k, _), (d2, ids) in zip(qs, outs)]
        res = []
        for k, Q in qs:
            chunks = [Q] if not batch else [Q[i:i + batch] for i in range(0, len(Q), batch)]
            parts = [merged(*engine.query(c, k), k) for c in chunks]
            res.append(parts[0] if len(parts) == 1 else
                       tuple(torch.cat([p[i] for p in parts]) for i in range(2)))
        return res

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev.device if args.backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def all_ranks(v: float) -> list:
        if world == 1:
            return [v]
        t = torch.tensor([v], dtype=torch.float64, device=dev.device if args.backend == "nccl" else "cpu")
        out = [torch.zeros_like(t) for _ in range(world)]
        torch.distributed.all_gather(out, t)
        return [float(x.item()) for x in out]

    # the clock sampler starts before the warm-up: nvidia-smi's start-up (NVML
    # init) contends with the driver, so it must be over -- with the GPU kept
    # busy, not idle -- before the timed region opens
    clk = Clocks(local, enabled=dev.cuda, period_ms=args.clock_ms).__enter__()
    from paper_2212_13297_b200 import _lib

    # (C3's 70 ms timed region -- 20 steps of 4 calls -- was an outlier in one run in three,
    # 50K-250K against 300K queries/s, always one stalled step among the first four
    # (SSB_BENCH_TRACE=1 prints the per-step host times).  Three things met there: the clock
    # sampler's sixth sample (0.5 s of settling = five periods: now re-armed at the region's
    # start), the profiler's lazy counter allocation inside its first launch (now done when
    # it is enabled) and the first routing probe of the region (every 16th lean call runs
    # the index stages).  What is left: that probe call still costs 5-8 ms instead of 3.3,
    # and 14-76 ms in two runs of ten.)
    prof_on = dev.cuda and not os.environ.get("SSB_BENCH_NOPROF")
    t_settle = time.perf_counter()
    for _ in range(args.warmup):
        step(Q_dev)
    while dev.cuda and time.perf_counter() - t_settle < 0.5:
        step(Q_dev)
    dev.sync()

    # ---- timed region (device-timed, max over ranks) -------------------------
    if dev.cuda:
        _lib.prof_enable(False)
        _lib.prof_reset()
        _lib.prof_enable(bool(prof_on))
        launches0 = _lib.launch_count()
    region = dev.region()
    try:
        barrier()
        dev.sync()
        clk.rearm()
        clk.mark()  # only the samples taken inside the region count
        region.start()
        step_s = []
        for _ in range(args.steps):
            t_step = time.perf_counter()
            step(Q_dev)
            step_s.append(time.perf_counter() - t_step)
        ms_local = region.stop()
        clk.sample_now()  # (after the region's closing event: a short region may hold no periodic sample)
        if os.environ.get("SSB_BENCH_TRACE"):
            print("[bench] host ms per timed step: " + " ".join(f"{1000 * x:.2f}" for x in step_s), file=sys.stderr)
        clk.mark()
        barrier()
    finally:
        clk.__exit__(None, None, None)
    prof, launches = {}, 0
    if dev.cuda:
        launches = _lib.launch_count() - launches0
        _lib.prof_enable(False)
        prof = _lib.prof_read()
    ms = max_over_ranks(ms_local)
    answers = sum(len(Q) for Q in cellq)
    value = answers * args.steps / (ms / 1000.0)
    # load balance: each rank's dominant-kernel time over the timed region
    top_name = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
    per_rank_ms = all_ranks(prof[top_name][0] if top_name else ms_local)

    # ---- e2e: the public API with host buffers, copies inside the region ------
    Q_host = [(k, dev.pinned(Q)) for k, Q in calls]
    h2d = sum(Q.numel() * 4 for _, Q in Q_host)
    d2h = sum(len(Q) * k * (4 + 8) for k, Q in calls)
    for _ in range(args.warmup):  # the host path's own warm-up (pinned uploads, result copies), untimed
        outs = step(Q_host)
        host = [(d2.cpu().numpy(), ids.cpu().numpy()) for d2, ids in outs]
    barrier()
    dev.sync()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        outs = step(Q_host)
        host = [(d2.cpu().numpy(), ids.cpu().numpy()) for d2, ids in outs]
    dev.sync()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = answers * args.steps / e2e_s

    # ---- single-query latency through the reference's own per-query API ------
    # (QueryEngine.exact_knn, query.py:296-348: one query per call, host
    # buffers, QueryStats included; N = 1 only -- a sharded query is a block)
    single = None
    if world == 1 and isinstance(engine, IndexEngine):
        from paper_2212_13297_b200 import QueryConfig

        k0, Q0 = calls[0]
        lat, routes = [], []
        for i in range(22):
            t0 = time.perf_counter()
            _, st = engine.engine.exact_knn(Q0[i % len(Q0)], QueryConfig(k=k0))
            if i >= 2:
                lat.append(time.perf_counter() - t0)
                routes.append(st.phase_reached)
        single = {"api": "QueryEngine.exact_knn (one query per call, host buffers)", "k": k0,
                  "median_ms": round(1000 * statistics.median(lat), 3), "p90_ms": round(
                      1000 * sorted(lat)[int(0.9 * len(lat))], 3), "calls": len(lat),
                  "phase_reached": sorted(set(routes))}

    # ---- parity (and, at N = 1, the CPU baseline) through the oracle ----------
    parity = cb = None
    if not args.no_cpu_baseline:
        threads = max(1, (os.cpu_count() or 1) // world)
        # the same sample on every rank: each rank's oracle answers over its
        # shard (global ids), merged like the GPU answers
        budget = args.cpu_seconds if world == 1 else args.cpu_seconds / 2
        sample = args.cpu_sample
        if world > 1 and not sample:
            sample = 2  # every rank must sample the same queries
        ans, secs = oracle_sample(wl, X, cellq, sample, budget, threads)
        if world > 1:
            from paper_2212_13297_b200.distributed import pack_keys, gather_keys, host_merge

            glob = []
            for c, j, k, od2, oid in ans:
                oid = np.where(oid >= 0, oid + lo, -1)
                keys = torch.from_numpy(pack_keys(od2[None, :], oid[None, :]))
                allk = gather_keys(keys.to(dev.device) if args.backend == "nccl" else keys)
                gd2, gid = host_merge(allk.cpu(), k)
                glob.append((c, j, k, gd2[0], gid[0]))
            ans = glob

        def gpu_rows(c, j):
            i, off = where[c]
            return host[i][0][off + j], host[i][1][off + j]

        parity = check_parity(ans, gpu_rows)
        if world == 1:
            cb = {"value": len(ans) / secs, "unit": "queries/s", "cores": threads, "kind": "port",
                  "cpu_model": cpu_model(),
                  "sample": f"{len(ans)} queries (round robin over the {len(wl.cells)} cells, about "
                            f"{args.cpu_seconds:.0f} s) of workload {wl.name} through the C oracle's exact scan "
                            f"(pscan.py:23-135 restated, {threads} threads); the same queries are the parity sample",
                  "build": ref_build_baseline(hi - lo, wl.n, wl.tau)}

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0 if not parity or parity["mismatches"] == 0 else 3

    # ---- roofline of the dominant kernel ---------------------------------------
    peaks = load_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    roof = None
    if top_name:
        kms, klaunch, kbytes, kflops = prof[top_name]
        avg_s = (kms / klaunch) / 1000.0
        long_region = ms >= 1000.0
        if kflops > 0:  # tensor-core kernel: FLOPs against the measured bf16 peak
            burst = float(peaks.get("bf16_tflops", 1590.0))
            sust = float(peaks.get("bf16_tflops_sustained", burst))
            tf_peak = sust if long_region else burst
            achieved = (kflops / klaunch) / avg_s / 1e12
            roof = {"kernel": top_name, "bound": "tensor", "achieved": round(achieved, 1), "peak": tf_peak,
                    "unit": "TFLOP/s", "frac": round(achieved / tf_peak, 4), "traffic": None,
                    "frac_vs_burst": round(achieved / burst, 4), "frac_vs_sustained": round(achieved / sust, 4),
                    "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained (timed region >= 1 s)" if long_region
                                    else "MEASURED_PEAKS.json bf16_tflops (burst; timed region < 1 s)")
                    if peaks else "fallback 1.59 PF",
                    # bf16 operand bytes the launch feeds the tensor cores (each row once per
                    # 256-query cluster) per second: NOT a DRAM rate (see traffic)
                    "operand_GBps": round((kbytes / klaunch) / avg_s / 1e9, 1)}
        else:
            achieved = (kbytes / klaunch) / avg_s / 1e9
            roof = {"kernel": top_name, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": None,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6.65 TB/s"}
        roof.update({"share_of_step": round(kms / ms, 4) if world == 1 else None,
                     "avg_launch_ms": round(kms / klaunch, 4)})
        # DRAM traffic per launch of this kernel from a committed `ncu --set full`
        # capture of the same workload (profiles/traffic.json), when there is one
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json"))).get(wl.name, {})
            if tr.get("kernel") == top_name:
                roof["traffic"] = tr["bytes_per_launch"]
                roof["traffic_source"] = tr["source"]
                roof["dram_GBps"] = round(tr["bytes_per_launch"] / avg_s / 1e9, 1)
        except (OSError, ValueError, KeyError):
            pass
    mean_ms = sum(per_rank_ms) / len(per_rank_ms)
    line = {
        "metric": "exact kNN queries/s", "value": round(value, 1), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: reference generator recipe (seeded Philox streams; see DESIGN.md Inputs)",
        "config": {"workload": wl.desc, "engine": getattr(engine, "name", type(engine).__name__),
                   "shards": world,
                   "calls_per_step": [{"k": k, "queries": len(Q)} for k, Q in calls],
                   "api": ("QueryEngine.knn_device_multi (ssb_query_multi: one host round trip per step)" if multi
                           else "QueryEngine.knn_device per call")
                   + ("; per-shard top-k packed on the device, NCCL all-gather + K-merge inside the step"
                      if world > 1 else ""),
                   "l2": "inputs larger than L2 (dataset %.2f GB > 126 MB)" % (N * wl.n * 4 / 1e9),
                   "data_gen_s": round(t_gen, 1)},
        "roofline": roof,
        "kernels": {k: {"ms": round(v[0], 3), "launches": v[1], "GB": round(v[2] / 1e9, 3),
                        "TFLOP": round(v[3] / 1e12, 3)} for k, v in prof.items()},
        "load_balance": {"kernel": top_name or "step", "ms_per_rank": [round(x, 3) for x in per_rank_ms],
                         "max_over_mean": round(max(per_rank_ms) / mean_ms, 4) if mean_ms > 0 else None},
        "parity": parity,
        "cpu_baseline": cb,
        "e2e": {"value": round(e2e, 1), "unit": "queries/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "single_query": single,
        "gpu_launches": launches,
        "build": dict(engine.build_info(hi - lo) or {}, **({"ingest": ingest} if ingest else {}),
                      **({"device_gen": device_gen} if device_gen else {})),
        "clocks": clk.summary(),
    }
    if comm:
        line["comm"] = comm
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    if parity and parity["mismatches"]:
        print(f"PARITY FAILURE: {parity['mismatches']} of {parity['checked']} sampled answers differ "
              f"from the oracle", file=sys.stderr)
        return 3
    return 0


def ingest_sample(args, X, wl):
    """file -> pinned double buffer -> HBM (ssb_ingest_file) on a sample of the
    shard written to a local file first (page cache: the pipeline, not the
    disk, is measured); a sample covering the whole shard becomes X_dev."""
    if args.ingest_gb <= 0:
        return None, None
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
    info = {"GBps": round(st["GBps"], 2), "bytes": st["bytes"], "rows": rows, "of_shard_rows": len(X),
            "source": "raw float32 file in the page cache, 64 MB pinned double buffer, "
                      f"{min(16, os.cpu_count() or 1)} read threads"}
    return (D if rows == len(X) else None), info


def device_gen_sample(args, X, wl, lo):
    """Device generator (documented Philox stream) on a sample of
    the shard size, beside the host generator."""
    import torch

    from paper_2212_13297_b200 import generate as _G

    g_rows = min(len(X), 4_000_000)
    g_fn = _G.unit_gaussian_device if wl.name == "c3" else _G.random_walks_device
    g_fn(1024, wl.n, 0)
    torch.cuda.synchronize()
    g0 = time.perf_counter()
    g_out = g_fn(g_rows, wl.n, 0, start=lo)
    torch.cuda.synchronize()
    g_s = time.perf_counter() - g0
    del g_out
    return {"series_per_s": round(g_rows / g_s, 1), "rows": g_rows}


if __name__ == "__main__":
    main()
