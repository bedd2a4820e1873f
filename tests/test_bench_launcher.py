"""bench.py --gpus N starts its own ranks (torch.distributed.run re-exec);
exercised on CPU with gloo: rank 0 prints one line with n_gpus = N and the
max over ranks."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [1, 2])
def test_bench_launcher_spawns_ranks(n):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--steps", "2",
                          "--launch-selftest"], capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["n_gpus"] == n and line["ranks_seen"] == n
    # the slowest rank sleeps 10 ms x n: the reported time is the max over ranks
    assert line["max_rank_seconds"] >= 0.01 * n - 1e-3
