"""The sharded executor across PROCESSES (not the in-process group): torchrun starts W ranks,
each runs the C++ executor on its block of every Dot/Conv and exchanges item ranges at the
executor's own gather points through hg_plan_set_gather_callback (gloo, host memory).  Every
rank's outputs must equal the reference's bit for bit, with the reference's profile counts.
On a one-GPU box the ranks share cuda:0; no device kernel waits on another rank (the exchange
is host-side after a stream synchronisation)."""
import json
import os
import socket
import subprocess
import sys

import pytest

from tests import golden_util as G

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,world", [("c1", 2), ("mini", 2), ("ops3", 3), ("pmodel_b", 2), ("c3_n2048", 2)])
def test_sharded_executor_across_processes(name, world, cuda_ok):
    if not os.path.exists(os.path.join(G.GOLDEN, f"net_{name}.json")):
        pytest.skip("golden missing")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "shard_proc.py"),
           name]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    res = [json.loads(ln[7:]) for ln in out.stdout.splitlines() if ln.startswith("RESULT ")]
    assert len(res) == world, out.stdout[-2000:]
    for r in res:
        assert r["counts_equal"], r
        assert r["gathers"], "no gather point was reached: the graph did not shard"
        for oid, o in r["outputs"].items():
            assert not o["bad"] and o["values_equal"], (r["rank"], oid, o)
