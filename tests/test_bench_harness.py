"""bench.py's multi-rank harness on CPU (gloo): `--gpus N` re-executes
itself under torchrun with one rank per (here: CPU) device, every rank holds
rows [rR/N, (r+1)R/N) of the config's table (strong scaling), the sharded
pipeline runs, the step time is the max over ranks, rank 0 prints one JSON
line with n_gpus = N."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
import bench  # noqa: E402


def test_shard_ranges_tile_the_table():
    for rows in (0, 1, 7, 1_470_000_000):
        for world in (1, 2, 3, 8):
            parts = [bench.shard_range(r, world, rows) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == rows
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))


def test_torchrun_argv():
    argv = bench.torchrun_argv(4, ["--gpus", "4"], 12345)
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in argv and "127.0.0.1" in argv and "12345" in argv


@pytest.mark.parametrize("gpus", [2, 3])
def test_dry_run_reports_n_ranks(gpus):
    env = {k: v for k, v in __import__("os").environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    proc = subprocess.run([sys.executable, str(REPO / "bench.py"), "--gpus", str(gpus),
                           "--dry-run", "--config", "c1", "--steps", "1", "--warmup", "0",
                           "--iterations", "3", "--dry-run-rows", "20000"],
                          cwd=REPO, env=env, capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stderr[-3000:]
    lines = [ln for ln in proc.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, proc.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == gpus and d["scaling"] == "strong" and d["dry_run"]
    assert d["shard"][0][0] == 0 and d["shard"][-1][1] == 20000
    assert d["graph"]["edges"] > 0
