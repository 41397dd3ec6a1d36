"""Throughput of the summarisation kernels (ssb_words, ssb_segment_stats) in
GB/s of row data read, against the measured HBM peak.  (GPU box)"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2212_13297_b200 import summarize as S

    N, n = 10_000_000, 256
    X = torch.randn(N, n, device="cuda", dtype=torch.float32)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json"))).get("hbm_gbs", 6542.4)
    starts = np.arange(16) * 16
    ends = starts + 16
    for name, fn in (("words", lambda: S.paa_words(X)), ("words+paa", lambda: S.paa_words(X, with_paa=True)),
                     ("segment_stats m=16", lambda: S.segment_stats_matrix(X, starts, ends)),
                     ("segment_stats m=16 overlapping",
                      lambda: S.segment_stats_matrix(X, starts // 2, ends)),
                     ("segment_stats m=1", lambda: S.segment_stats_matrix(X, np.array([0]), np.array([n]))),
                     ("segment_stats m=4", lambda: S.segment_stats_matrix(X, np.arange(4) * 64, np.arange(1, 5) * 64))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        gbs = N * n * 4 / ms / 1e6
        print(json.dumps({"kernel": name, "ms": round(ms, 3), "GBps": round(gbs, 1), "frac": round(gbs / peak, 3)}))


if __name__ == "__main__":
    main()
