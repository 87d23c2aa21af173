"""bench.py's launch contract on CPU: `--gpus N` without a torchrun
environment spawns N ranks itself, and the rank-0 line carries every rank's
step time (the timing/reduction plumbing of the real run, over gloo, with a
no-op step)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=240, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_gpus_flag_spawns_ranks():
    line = _run(["--dry-run", "--gpus", "2", "--steps", "2"])
    assert line["n_gpus"] == 2
    assert len(line["per_rank_ms"]) == 2
    assert line["ms_per_step"] == max(line["per_rank_ms"])


def test_single_rank_default():
    line = _run(["--dry-run", "--steps", "1"])
    assert line["n_gpus"] == 1 and len(line["per_rank_ms"]) == 1
