"""Drop-in proof: the UNMODIFIED reference executor (heg::execute) run over the
reference CkksBackend and over GpuCkksBackend (integration/gpu_ckks_backend.hpp,
every op through include/hegpu.h on the B200) must give bit-identical outputs
and identical ExecProfile counts.  The binary is built from the reference
headers where they exist (build() here) and travels to the GPU box."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "drop_in_test")


@pytest.mark.parametrize("name", ["mini", "c1"])
def test_reference_executor_over_gpu_backend(name, cuda_ok):
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/drop_in_test not built (needs the reference headers at build time)")
    from paper_1810_10121_b200 import graphs

    spec = graphs.GOLDEN_NETS[name]
    g, x, ctxp = graphs.build(spec)
    with tempfile.TemporaryDirectory() as d:
        gp, xp = os.path.join(d, "g.json"), os.path.join(d, "x.f64")
        with open(gp, "w") as f:
            json.dump(g, f)
        x.astype(np.float64).tofile(xp)
        out = subprocess.run([BIN, gp, xp, str(spec["batch"]), str(ctxp["n"]), str(ctxp["scale_bits"]),
                              ",".join(map(str, ctxp["bits"])), str(ctxp["security"]), str(spec["key_seed"]),
                              str(spec["exec_seed"])], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["outputs_bit_equal"] and res["profile_counts_equal"], res
