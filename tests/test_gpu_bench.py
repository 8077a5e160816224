"""``bench.py --gpus 2`` launches itself (torchrun, 2 ranks) and prints one
rank-0 line with n_gpus == 2, the per-rank spread and the handoff object.
Runs in SZ_BENCH_BACKEND=gloo test mode so both ranks share the one GPU of
the test box (time-sliced: the numbers are not a measurement)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_bench_self_launches_two_ranks():
    env = dict(os.environ, SZ_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--elements", str(1 << 24), "--e2e-steps", "1"]
    res = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    assert line["config"]["elements_override"] == 1 << 24
    assert line["per_rank_gbs"]["min"] <= line["per_rank_gbs"]["max"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    ho = line["handoff"]
    assert "error" not in ho, ho
    for tag in ("realistic_eps0.16", "escape_heavy_eps7.89"):
        assert ho[tag]["bitexact"] is True, ho
