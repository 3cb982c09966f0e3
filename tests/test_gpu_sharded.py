"""Multi-rank GPU parity of the position-sharded path through the
C-ABI, against the fp64 oracle: the fused device-side exchange with W logical ranks in one
process, and with one process per rank (2 ranks sharing this box's GPU) for both the fused
exchange and the torch.distributed-collective path.  Each case runs in a subprocess under a
timeout (tests/sharded_worker.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=420, env_extra=None):
    env = dict(os.environ)
    # one hardware queue per stream, so a rank's stream waiting on its peers never blocks
    # another rank's stream behind it (logical ranks in one process)
    env["CUDA_DEVICE_MAX_CONNECTIONS"] = "32"
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("{")][-1]
    return json.loads(line)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("W,extra", [(2, []), (3, []), (4, []), (2, ["--cyclic"]), (3, ["--cyclic", "--n", "3990"]),
                                     (2, ["--vonly", "--prefetch"]), (3, ["--cyclic", "--prefetch"]),
                                     (2, ["--dtype", "fp32", "--n", "1003"]), (3, ["--norm", "1"]), (8, ["--n", "8000", "--requests", "1"])])
def test_fused_exchange_logical_ranks(W, extra):
    r = _run(["-m", "tests.sharded_worker", "logical", "--W", str(W), *extra])
    assert r["layers"] > 0 and r["max_out_rel"] < (1e-4 if "fp32" in extra else 2e-2), r


def test_fused_exchange_in_cuda_graphs():
    # the whole sharded request of every rank captured in one CUDA graph per rank, replayed
    # concurrently: the exchange's put / wait kernels are ordinary graph nodes
    r = _run(["-m", "tests.sharded_worker", "logical", "--W", "3", "--graph", "--cyclic"])
    assert r["graph"] is True and r["max_out_rel"] < 2e-2, r


@pytest.mark.parametrize("impl,extra", [("fused", []), ("fused", ["--cyclic", "--prefetch"]), ("collective", []),
                                        ("collective", ["--cyclic"])])
def test_two_processes_one_gpu(impl, extra):
    r = _run(["-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr=127.0.0.1",
              f"--master-port={_free_port()}", "-m", "tests.sharded_worker", "mp", "--impl", impl, *extra])
    assert r["W"] == 2 and r["layers"] > 0 and r["max_out_rel"] < 2e-2, r
