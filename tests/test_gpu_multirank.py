"""bench.py's sharded cfg5 path under torchrun with two ranks (on one GPU when
the box has one: the ranks share nothing but gloo barriers, no kernel waits
on another rank), against a single-rank run: the shards each rank dumps,
concatenated, must equal the single run bit for bit, and both must carry the
JSON contract of a strong-scaling split."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--workload", "cfg2", "--ns", "4", "--rows", "65536", "--workloads", "cfg5", "--cfg5-rows", str(1 << 20),
        "--steps", "1", "--warmup", "3", "--reps", "6", "--no-e2e", "--no-cpu"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(cmd, tmp):
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
    return json.loads(line)


def test_cfg5_two_ranks_equal_single(tmp_path):
    one = tmp_path / "one"
    two = tmp_path / "two"
    j1 = _run([sys.executable, "bench.py", *ARGS, "--dump-dir", str(one)], one)
    j2 = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2", *ARGS,
               "--dump-dir", str(two)], two)
    assert j2["n_gpus"] == 2 and j1["n_gpus"] == 1
    b1, b2 = j1["workloads"]["cfg5"], j2["workloads"]["cfg5"]
    assert b2["scaling"] == "strong" and b2["arrays_total"] == b1["arrays_total"] == 1 << 20
    assert len(b2["gbs_per_gpu"]) == 2 and b2["arrays_per_gpu"] == (1 << 20) // 2
    full = np.load(one / "cfg5_rank0.npy")
    parts, lo_next = [], 0
    for r in range(2):
        meta = json.loads((two / f"cfg5_rank{r}.json").read_text())
        assert meta["lo"] == lo_next
        lo_next = meta["hi"]
        parts.append(np.load(two / f"cfg5_rank{r}.npy"))
    assert lo_next == 1 << 20
    assert np.array_equal(np.concatenate(parts, axis=1), full)
