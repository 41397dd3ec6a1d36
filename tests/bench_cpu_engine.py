"""CPU stand-in engine for the bench.py plumbing tests (no GPU here).

bench.py loads it only when SSB_BENCH_TEST_ENGINE=bench_cpu_engine:OracleEngine
is set (tests/test_bench_cpu.py): the shard search is the oracle's exact scan
(test infrastructure), so the multi-rank launch, the all-gather + merge inside
the timed step, max-over-ranks timing, the parity check and the JSON line are
exercised on CPU with the gloo backend."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))


class OracleEngine:
    name = "test engine: oracle exact scan per shard (CPU, gloo)"

    def __init__(self, X, tau, id_base=0, **_):
        self.X = X.numpy() if hasattr(X, "numpy") else np.asarray(X)
        self.id_base = id_base

    @staticmethod
    def merge_fn(all_keys, k):
        import torch

        from paper_2212_13297_b200.distributed import host_merge

        d2, ids = host_merge(all_keys, k)
        return torch.from_numpy(d2), torch.from_numpy(ids)

    def build_info(self, N):
        return {"series_per_s": None, "note": "test engine: no build"}

    def query(self, Q, k):
        import oracle
        import torch

        d2, ids = oracle.knn_scan(self.X, Q.numpy(), k)
        ids = np.where(ids >= 0, ids + self.id_base, -1)
        return torch.from_numpy(d2), torch.from_numpy(ids)
