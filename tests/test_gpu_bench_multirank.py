"""bench.py's multi-rank path (torchrun, one process per GPU, chain shards
with chain_offset = rank * m, the global stop rule, ESS partials all-reduced,
max-over-ranks timing) exercised on a one-GPU box: both ranks on cuda:0 with
gloo collectives (--one-device).  A functional check of the code path the
driver's 2/4/8-GPU runs take; its timings say nothing about scaling."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("config", ["c2", "c3"])
def test_bench_runs_two_ranks(config):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py",
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--config", config, "--chains", "2048",
           "--samples", "60", "--no-cpu", "--one-device"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["chains_total"] == 4096
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["ess_pooled"] is not None and d["rhat_max"] is not None
