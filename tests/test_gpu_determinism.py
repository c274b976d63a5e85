"""Repeated runs of the same plan must give identical ciphertexts at every node.
A race (e.g. a kernel reading shared memory before it is staged) shows up as
run-to-run differences long before it fails a golden comparison."""
import hashlib
import os

import pytest

from tests import golden_util as G

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,reps", [("c4_n2048", 3), ("c5", 3)])
def test_every_node_is_deterministic(name, reps, cuda_ok):
    import paper_1810_10121_b200 as P
    from paper_1810_10121_b200 import graphs

    if not os.path.exists(os.path.join(G.GOLDEN, f"net_{name}.json")):
        pytest.skip("golden spec not present")
    spec = graphs.GOLDEN_NETS[name]
    g, x, ctxp = graphs.build(spec)
    g = dict(g)
    g["outputs"] = [n["id"] for n in g["nodes"] if n["op"] not in ("Constant", "Parameter")]
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
    plan.bind_input("x", x)
    first = None
    for _ in range(reps):
        plan.run()
        d = {}
        for oid in g["outputs"]:
            try:
                d[oid] = hashlib.sha256(plan.output_ciphertexts(oid).tobytes()).hexdigest()
            except P.HEError:  # a node that stays plaintext (constant folding)
                pass
        if first is None:
            first = d
        else:
            diff = [k for k in d if d[k] != first[k]]
            assert not diff, f"{name}: nodes {diff} differ between runs"
    plan.close()
