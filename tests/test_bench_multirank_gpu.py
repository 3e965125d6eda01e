"""The bench's N>1 path (torchrun, one rank per GPU, hash-sharded store,
keyframe broadcast, max-over-ranks timing) run end to end with two ranks
sharing the one GPU of this run over gloo -- a functional check of the
multi-rank code path (replicated and routed footprints), not a measurement."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("route", ["0", "1"])
def test_bench_two_ranks_one_gpu(route):
    env = dict(os.environ, RF_DIST_BACKEND="gloo", RF_ROUTE=route,
               RF_BENCH_BLOCKS="700000")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(REPO, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--keyframes", "40", "--no-cpu-baseline", "--no-e2e"]
    out = subprocess.run(cmd, cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
    assert "hash-sharded x2" in d["config"]["parallelism"]
    assert ("routed" in d["config"]["parallelism"]) == (route == "1")
