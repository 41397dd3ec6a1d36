"""bench.py contract pieces that run without a GPU: the reference arm (the
oracle port on host cores) prints one JSON line with the contract keys."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "c1", "--rows", "20000", "--steps", "1", "--warmup", "0",
                          "--cpu-sample", "2"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    j = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["value"] > 0 and j["unit"] == "queries/s"
    assert j["cpu_baseline"]["kind"] == "port" and j["cpu_baseline"]["cores"] >= 1
    assert j["e2e"]["h2d_bytes_per_step"] == 0 and j["e2e"]["value"] == j["value"]


def test_gpus_2_spawns_two_ranks_and_merges():
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself under
    torch.distributed.run with two ranks (gloo here); rank 0 prints ONE line
    with n_gpus 2, the communicator's rank count, the per-rank load balance and
    a green parity check of the merged (all-gathered) answers."""
    env = dict(os.environ, SSB_BENCH_TEST_ENGINE="bench_cpu_engine:OracleEngine")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                          "--workload", "c2", "--rows", "6000", "--queries", "6", "--steps", "2", "--warmup", "1",
                          "--cpu-sample", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["comm"]["nranks"] == 2 and j["comm"]["allreduce_ranks"] == 2
    assert len(j["load_balance"]["ms_per_rank"]) == 2
    assert j["parity"]["checked"] == 3 * 6 and j["parity"]["mismatches"] == 0
    assert j["value"] > 0 and j["e2e"]["value"] > 0 and "merge" in j["config"]["api"] or "K-merge" in j["config"]["api"]
