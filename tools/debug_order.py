"""Diagnostic: per-node ciphertext digests of one golden net, run fresh or after other nets
in the same process (isolates state carried between plans/contexts)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1810_10121_b200 as P  # noqa: E402
from paper_1810_10121_b200 import graphs  # noqa: E402


def run(name, all_nodes=True):
    spec = graphs.GOLDEN_NETS[name]
    g, x, ctxp = graphs.build(spec)
    if all_nodes:
        g = dict(g)
        g["outputs"] = [n["id"] for n in g["nodes"] if n["op"] not in ("Constant", "Parameter")]
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
    plan.bind_input("x", x)
    plan.run()
    out = {}
    for oid in g["outputs"]:
        try:
            w = plan.output_ciphertexts(oid)
            out[oid] = hashlib.sha256(w.tobytes()).hexdigest()[:16]
        except Exception as e:
            out[oid] = f"err {e}"
    plan.close()
    return out


target = sys.argv[1]
pre = sys.argv[2:]
for p in pre:
    run(p, all_nodes=False)
print(json.dumps(run(target)))
