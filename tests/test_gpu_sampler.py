"""The counter-based GPU sampler must reproduce the reference's sequential
splitmix64 + Box-Muller streams exactly (poly.hpp:257-276, common.hpp:100-105),
including the host fix-up path for values near a rounding boundary."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1810_10121_b200 as P
n, items = int(sys.argv[1]), int(sys.argv[2])
ctx = P.Context(n, [30, 30, 30], 30, security=0)
seeds = np.random.default_rng(7).integers(0, 2**63, items, dtype=np.uint64)
seeds[0] = 0; seeds[1] = 2**64 - 1
out = torch.zeros(items * 3 * n, dtype=torch.int64, device="cuda")
P.call("hg_sample_encryption", ctx, seeds.ctypes.data_as(P.u64p), items, out)
host = np.zeros(items * 3 * n, dtype=np.int64)
P.call("hg_sample_encryption_host", ctx, seeds.ctypes.data_as(P.u64p), items, host.ctypes.data)
got = out.cpu().numpy()
assert np.array_equal(got, host), np.nonzero(got != host)[0][:10]
u = host.reshape(items, 3, n)
assert set(np.unique(u[:, 0])) <= {-1, 0, 1}
print("sampler ok", np.abs(u[:, 1:]).max())
""" % ROOT


@pytest.mark.parametrize("guard", [None, "0.01"])
def test_gpu_sampler_matches_host(cuda_ok, guard):
    env = dict(os.environ)
    if guard:
        env["HG_SAMPLER_GUARD"] = guard  # widen the fix-up band so the host path runs many times
    out = subprocess.run([sys.executable, "-c", SCRIPT, "4096", "24"], capture_output=True, text=True, env=env,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "sampler ok" in out.stdout
