"""Diagnostic: run a golden net R times in one process (all nodes as outputs) and report
per-node digest disagreements across runs (catches nondeterminism / races)."""
import collections
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1810_10121_b200 as P  # noqa: E402
from paper_1810_10121_b200 import graphs  # noqa: E402

name, reps = sys.argv[1], int(sys.argv[2])
spec = graphs.GOLDEN_NETS[name]
g, x, ctxp = graphs.build(spec)
g = dict(g)
g["outputs"] = [n["id"] for n in g["nodes"] if n["op"] not in ("Constant", "Parameter")]
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
seen = collections.defaultdict(collections.Counter)
fresh = os.environ.get("FRESH_PLAN") == "1"
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
plan.bind_input("x", x)
for r in range(reps):
    if fresh:
        plan.close()
        plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
        plan.bind_input("x", x)
    plan.run()
    for oid in g["outputs"]:
        try:
            seen[oid][hashlib.sha256(plan.output_ciphertexts(oid).tobytes()).hexdigest()[:12]] += 1
        except P.HEError:  # plaintext-valued node
            pass
bad = {k: dict(v) for k, v in seen.items() if len(v) > 1}
print(json.dumps({"net": name, "reps": reps, "nondeterministic_nodes": bad}))
