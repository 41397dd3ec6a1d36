"""Time the REFERENCE index build (pure Python, /root/reference) on this
container's host cores -- the CPU build baseline bench.py reports beside the
GPU build (build series/s measured at <= 1M, then
extrapolated).  The reference cannot travel to the GPU box (it is not
installed there), so its measurement is committed:

    python tools/ref_build_probe.py --rows 100000 --tau 1000 >> profiles/ref_build_cpu.jsonl

Runs build_index(dataset file, settings, num_threads=cores) exactly as the
reference's own callers do (build.py:363-458), on the reference generator's
dataset (generate.py:42-55, seed 0).
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=100_000)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--tau", type=int, default=1000)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 2)
    ap.add_argument("--reference", default="/root/reference/pkg/src")
    a = ap.parse_args()
    sys.path.insert(0, a.reference)
    from seriesearch import build as rbuild
    from seriesearch import generate as rgen
    from seriesearch import persist as rpersist

    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "data.bin")
        t0 = time.perf_counter()
        rgen.generate_random_walk(a.rows, a.n, 0, path)
        t_gen = time.perf_counter() - t0
        s = rpersist.IndexSettings(series_length=a.n, dataset_size=a.rows, leaf_threshold=a.tau)
        t0 = time.perf_counter()
        idx = rbuild.build_index(path, s, num_threads=max(2, a.threads))
        t_build = time.perf_counter() - t0
        leaves = sum(1 for _ in idx.root.iter_leaves()) if hasattr(idx, "root") else None
    print(json.dumps({"what": "reference build_index (build.py:363-458), pure Python",
                      "rows": a.rows, "n": a.n, "tau": a.tau, "num_threads": max(2, a.threads),
                      "build_s": round(t_build, 2), "series_per_s": round(a.rows / t_build, 1),
                      "leaves": leaves, "gen_s": round(t_gen, 1), "cores": os.cpu_count(),
                      "cpu_model": cpu_model(), "python": platform.python_version(),
                      "host": "builder container (the reference is not installed on the GPU box)"}))


if __name__ == "__main__":
    main()
