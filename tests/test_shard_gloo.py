"""World-size-2 (and 3) CPU check of the multi-GPU path's host logic over gloo:
the executor's partition rule (hg_shard_partition, read through the C-ABI),
the shard-preserving ops and the all-gather schedule (in-place broadcasts of
each rank's ranges) reproduce the unsharded result exactly on every rank.
See tests/shard_model.py; tests/test_gpu_shard.py runs the same rules on the GPU."""
import json
import os
import socket
import subprocess
import sys

import pytest

from tests.shard_model import coalesce

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_covers_every_output_once():
    import paper_1810_10121_b200 as P

    for groups, mg in [(1, 16), (1, 100), (1, 3), (169, 5), (256, 32), (2, 7), (7, 1), (0, 4), (4, 0)]:
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                g0, g1, m0, m1 = P.shard_partition(groups, mg, world, r)
                assert 0 <= g0 <= g1 <= groups and 0 <= m0 <= m1 <= mg
                seen += [(g, m) for g in range(g0, g1) for m in range(m0, m1)]
            assert sorted(seen) == [(g, m) for g in range(groups) for m in range(mg)], (groups, mg, world)
            sizes = [(lambda b: (b[1] - b[0]) * (b[3] - b[2]))(P.shard_partition(groups, mg, world, r))
                     for r in range(world)]
            if groups * mg:
                assert max(sizes) - min(sizes) <= max(mg if groups > 1 else 1, 1), (groups, mg, world, sizes)


def test_coalesce():
    assert coalesce([5, 1, 2, 3, 9, 10]) == [(1, 4), (5, 6), (9, 11)]


@pytest.mark.parametrize("graph,world", [("c3", 2), ("mlp", 2), ("mlp", 3)])
def test_sharded_graph_over_gloo(graph, world):
    port = _port()
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "shard_model.py"), "--rank", str(r),
                               "--world", str(world), "--port", str(port), "--graph", graph],
                              cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(world)]
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            p.kill()
            raise
        assert p.returncode == 0, e[-3000:] + o
        outs.append(json.loads(o.strip().splitlines()[-1]))
    assert all(o["ok"] for o in outs)
    assert all(o["gathers"] >= 1 for o in outs)
