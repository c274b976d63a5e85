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


def _run(args, timeout=900):
    out = subprocess.run([BIN] + [str(a) for a in args], capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stdout + out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def _need_bin():
    if not os.path.exists(BIN):
        pytest.skip("integration/_build/drop_in_test not built (needs the reference headers at build time)")


# every paradigm: EncryptedData (mini, c1), EncryptedModel / EncryptedBoth (pmodel_m, pmodel_b, mini_b:
# ct x ct contractions through the adapter's weighted_sum_cipher override, ckks_backend.hpp:413-450)
@pytest.mark.parametrize("name", ["mini", "c1", "pmodel_m", "pmodel_b", "mini_b"])
def test_reference_executor_over_gpu_backend(name, cuda_ok):
    _need_bin()
    from paper_1810_10121_b200 import graphs

    spec = graphs.GOLDEN_NETS[name]
    g, x, ctxp = graphs.build(spec)
    with tempfile.TemporaryDirectory() as d:
        gp, xp = os.path.join(d, "g.json"), os.path.join(d, "x.f64")
        with open(gp, "w") as f:
            json.dump(g, f)
        x.astype(np.float64).tofile(xp)
        args = [gp, xp, spec["batch"], ctxp["n"], ctxp["scale_bits"], ",".join(map(str, ctxp["bits"])),
                ctxp["security"], spec["key_seed"], spec["exec_seed"]]
        if "paradigm" in spec:
            args.append(f"--paradigm={spec['paradigm']}")
        res = _run(args)
    assert res["outputs_bit_equal"] and res["profile_counts_equal"], res


# size-generic primitives (ckks_backend.hpp:261-297, 556-578): size-3 operands, unequal-size
# add/sub, 3x2 products (size 4, no relin), and the single-relin weighted_sum_cipher
@pytest.mark.parametrize("ring", [(2048, 30, [45, 30, 30, 45]), (4096, 26, [36, 26, 26, 36])])
def test_size_generic_primitives(ring, cuda_ok):
    _need_bin()
    n, sb, bits = ring
    res = _run(["ops", n, sb, ",".join(map(str, bits)), 41])
    assert res["all_equal"], res


# bench_gemm / bench_network (bench.hpp:75-127) take an HEBackend&: over the GPU adapter their
# rows carry the reference's bypass counts, and the gemm graphs' outputs are bit-identical
def test_bench_gemm_and_network_over_gpu_backend(cuda_ok):
    _need_bin()
    from paper_1810_10121_b200 import graphs

    spec = graphs.GOLDEN_NETS["mini"]
    g, _, ctxp = graphs.build(spec)
    with tempfile.TemporaryDirectory() as d:
        gp = os.path.join(d, "g.json")
        with open(gp, "w") as f:
            json.dump(g, f)
        res = _run(["bench", 6, gp, 8, ctxp["n"], ctxp["scale_bits"], ",".join(map(str, ctxp["bits"])), 3])
    assert res["bypass_counts_equal"] and res["gemm_outputs_bit_equal"], res
    assert [r["bypass"] for r in res["gpu_gemm_rows"]] == [r["bypass"] for r in res["ref_gemm_rows"]]
