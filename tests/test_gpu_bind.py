"""Input binding (hg_plan_bind_input: pack_cipher = encode + encrypt per column, packing.hpp:85-102,
ckks_backend.hpp:182-236) as the chunked pipeline: pageable host, pinned host and device inputs give
the reference's ciphertexts (the net goldens), re-binding rewrites the buffers in place, and an
encoder overflow is a validation error that leaves the parameter unbound."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _plan(name):
    import paper_1810_10121_b200 as P
    from paper_1810_10121_b200 import graphs
    from tests import golden_util as G

    gold = G.load_net(name)
    spec = gold["spec"]
    graph, x, ctxp = graphs.build(spec)
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, graph, spec["batch"], spec["exec_seed"])
    return P, G, gold, plan, x, (ctx, keys)


def _check(G, gold, plan):
    plan.run()
    for oid, want in gold["outputs"].items():
        assert G.sha(plan.output(oid)) == want["values_sha256"], oid


# c3_n2048 binds 784 columns (three chunks of the pipeline); mini binds fewer than one chunk
@pytest.mark.parametrize("name", ["c3_n2048", "mini"])
def test_bind_sources_give_the_golden_outputs(name, cuda_ok):
    import torch

    P, G, gold, plan, x, _keep = _plan(name)
    x = np.ascontiguousarray(x, dtype=np.float64)
    plan.bind_input("x", x)  # pageable host memory
    _check(G, gold, plan)
    plan.bind_input("x", torch.from_numpy(x).pin_memory())  # pinned host memory, re-bound in place
    _check(G, gold, plan)
    plan.bind_input("x", torch.from_numpy(x).cuda())  # device memory (one chunk, no copy)
    _check(G, gold, plan)
    # a different batch in between must not leave anything behind
    plan.bind_input("x", np.ascontiguousarray(x[::-1]))
    plan.run()
    plan.bind_input("x", x)
    _check(G, gold, plan)


def test_bind_overflow_unbinds_the_parameter(cuda_ok):
    P, G, gold, plan, x, _keep = _plan("mini")
    x = np.ascontiguousarray(x, dtype=np.float64)
    plan.bind_input("x", x)
    _check(G, gold, plan)
    with pytest.raises(P.HEError) as ei:
        plan.bind_input("x", x * 1e18 + 1e18)
    assert ei.value.category == "validation" and "overflows" in str(ei.value)
    with pytest.raises(P.HEError) as ei:
        plan.run()
    assert "no input bound" in str(ei.value)
    plan.bind_input("x", x)
    _check(G, gold, plan)
