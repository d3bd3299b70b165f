"""bench.py's multi-rank plumbing on CPU (gloo): `--gpus N` without torchrun starts the N
ranks itself, the global batch of N x batch_per_gpu sequences is sharded by
shard.shard_range, every sequence's final row is gathered to rank 0 in global order, and
the step time is the max over ranks.  The real arm runs the same code path
with the CUDA engine over NCCL (`--impl stub` swaps only the engine)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [1, 2, 3])
def test_bench_spawns_ranks_and_gathers_in_order(n):
    r = subprocess.run([sys.executable, BENCH, "--impl", "stub", "--gpus", str(n), "--steps", "2", "--warmup", "1"],
                       capture_output=True, text=True, timeout=300, env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == n
    B = d["config"]["batch_per_gpu"]
    assert d["config"]["global_batch"] == n * B
    assert d["gathered_last_col"] == [float(i) for i in range(n * B)]
    assert d["local_sequences"] == list(range(B))  # rank 0's shard
    assert d["ms_per_step"] > 0


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, BENCH, "--impl", "stub", "--gpus", "1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=120, env=env)
    assert r.returncode != 0 and "does not match WORLD_SIZE" in r.stderr
