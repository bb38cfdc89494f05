"""bench.py's N > 1 path on a one-GPU box: two and three ranks share cuda:0 over
gloo (GWN_BENCH_ONE_GPU=1 test hook), and rank 0 checks that the sharded,
packed and all-gathered results equal one full evaluation bit for bit
(SURVEY §8(e)).  The timings of such a run are meaningless and never reported."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_bench_sharded_gather_equals_full_eval(world):
    env = dict(os.environ, GWN_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(_port()), os.path.join(REPO, "bench.py"), "--gpus", str(world), "--steps", "3",
           "--warmup", "3", "--config", "2", "--no-extras", "--no-cpu-baseline",
           "--queries", "65537"]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "one-gpu gather check: identical" in r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == world and line["config"]["queries"] == 65537 * world
