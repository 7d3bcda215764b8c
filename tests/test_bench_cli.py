"""bench.py plumbing on CPU (no GPU): `--gpus N` without torchrun launches N
ranks itself (torch.distributed.run on 127.0.0.1) and rank 0 prints one
line reporting n_gpus = N; the --dry-run mode does the multi-rank setup
(z-slab partition + halo plan through gloo collectives) without measuring."""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


@pytest.mark.parametrize("n", [2, 3])
def test_bench_spawns_ranks_on_cpu(n):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(n), "--dry-run"],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["dry_run"] is True and d["value"] is None
    rows = d["config"]["ranks_rows"]
    assert rows[0] == 0 and rows[-1] == 400 ** 3 and len(rows) == n + 1
    assert all(r % (400 * 400) == 0 for r in rows)  # whole z-planes per rank
    assert d["config"]["max_halo_send"] == 2 * 400 * 400 if n > 2 else 400 * 400
