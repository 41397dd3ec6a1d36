"""Streamed file scan on the GPU box (pscan.pscan / scan_file, csrc/ingest.cu):
writes a dataset file of device-generated random walks, then times the
streamed exact k-NN over it for several query-block sizes, beside the plain
file -> HBM ingest (the same read + copy pipeline without the scan: the
pipeline's ceiling) and a parity check of a few answers against the resident
brute-force scan (itself bit-exact vs the oracle in the tests).

    python tools/scan_file_probe.py --rows 8000000 --blocks 1,16,128,1000

Prints one JSON line per measurement.
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=8_000_000)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--blocks", default="1,16,128,1000")
    ap.add_argument("--chunk-mb", type=int, default=256)
    ap.add_argument("--dir", default=tempfile.gettempdir())
    a = ap.parse_args()
    import numpy as np
    import torch

    from paper_2212_13297_b200 import generate, ingest_file, knn_batch, scan_file

    path = os.path.join(a.dir, f"ssb_scan_probe_{a.rows}x{a.n}.bin")
    t0 = time.perf_counter()
    with open(path, "wb") as f:
        step = 1 << 20
        for s in range(0, a.rows, step):
            c = min(step, a.rows - s)
            f.write(generate.random_walks_device(c, a.n, 0, start=s).cpu().numpy().tobytes())
    print(json.dumps({"write_file_s": round(time.perf_counter() - t0, 2), "GB": round(a.rows * a.n * 4 / 1e9, 2)}),
          flush=True)
    cb = a.chunk_mb << 20
    for rep in range(2):
        X, st = ingest_file(path, a.n, chunk_bytes=cb)
        print(json.dumps({"what": "ingest", "rep": rep, "GBps": round(st["GBps"], 2), "s": round(st["seconds"], 3)}),
              flush=True)
    Xd = X
    Qs = generate.random_walks_device(max(int(b) for b in a.blocks.split(",")), a.n, 1)
    for b in (int(v) for v in a.blocks.split(",")):
        Q = Qs[:b]
        for rep in range(2):
            d2, ids, st = scan_file(path, a.n, Q, a.k, chunk_bytes=cb)
            torch.cuda.synchronize()
            line = {"what": "scan_file", "B": b, "k": a.k, "rep": rep, "chunks": st["chunks"],
                    "s": round(st["seconds"], 3), "GBps": round(st["GBps"], 2),
                    "queries_per_s": round(b / st["seconds"], 2)}
            if rep == 1:
                rd2, rids = knn_batch(Xd, Q[:4], a.k)
                line["parity_vs_resident_scan"] = bool(torch.equal(rids, ids[:4]) and
                                                       torch.equal(rd2.view(torch.int32), d2[:4].view(torch.int32)))
            print(json.dumps(line), flush=True)
    del Xd, X
    os.remove(path)


if __name__ == "__main__":
    main()
