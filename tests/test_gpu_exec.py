"""GPU graph executor vs the reference executor (heg::execute + CkksBackend).

Golden fixtures come from the unmodified reference run on the same JSON graph,
keys seed, input tensor and exec seed (tests/golden/make_golden.py nets).  Every
output ciphertext must match bit for bit in the coefficient domain, decoded
outputs must match bit for bit, and the ExecProfile counts must be identical."""
import os

import numpy as np
import pytest

from tests import golden_util as G

pytestmark = pytest.mark.gpu

NETS = ["mini", "mini_nb", "ops2", "ops3", "ops3_na", "pmodel_m", "pmodel_b", "mini_b", "wide_p20", "wide_p56", "wide_p60", "c1", "c3_n2048",
        "c5_n2048", "c4_n2048", "c4s", "c3", "c5", "c4"]


def _available(name):
    return os.path.exists(os.path.join(G.GOLDEN, f"net_{name}.json"))


@pytest.mark.parametrize("name", [n for n in NETS if _available(n)])
def test_net_bit_exact(name, cuda_ok):
    import torch

    import paper_1810_10121_b200 as P
    from paper_1810_10121_b200 import graphs

    gold = G.load_net(name)
    spec = gold["spec"]
    graph, x, ctxp = graphs.build(spec)
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, graph, spec["batch"], spec["exec_seed"])
    if "paradigm" in spec or "bypass" in spec:
        plan.set_options(paradigm=spec.get("paradigm"), bypass=spec.get("bypass"))
    plan.bind_input("x", x)
    plan.run()
    prof = plan.profile()
    ref = gold["profile"]
    assert prof["bypass"] == ref["bypass"], (prof["bypass"], ref["bypass"])
    assert prof["ct_ops"] == ref["ct_ops"], (prof["ct_ops"], ref["ct_ops"])
    assert prof["peak_elements"] == ref["peak_elements"]
    for oid, want in gold["outputs"].items():
        elems, level, scale = plan.output_info(oid)
        assert elems == len(want["elements"])
        assert level == want["elements"][0]["level"]
        assert scale == want["elements"][0]["scale"], (scale, want["elements"][0]["scale"])
        words = plan.output_ciphertexts(oid)
        d = torch.from_numpy(words.view(np.int64)).cuda()
        P.ntt(ctx, d, elems * 2 * (level + 1), level + 1, inverse=True)
        coeff = d.cpu().numpy().view(np.uint64).reshape(elems, -1)
        bad = [e for e in range(elems) if G.sha(coeff[e]) != want["ct_sha256"][e]]
        assert not bad, f"{name}/{oid}: ciphertexts {bad[:8]} differ from the reference"
        vals = plan.output(oid)
        assert G.sha(vals) == want["values_sha256"], f"{name}/{oid}: decoded values differ"
        # the pipelined output path (decode on a host thread) returns the same doubles
        assert G.sha(plan.output_async(oid).wait()) == want["values_sha256"]
    plan.close()
