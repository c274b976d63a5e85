"""Per-phase host timing of the bench's pipelined e2e loop (bind / run / output_async / wait)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(os.environ.get("ITERS", "20"))
spec, g, x, ctxp = bench.build_workload(config, 4096 if config in ("c1", "c3") else 8192)
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
xh = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).pin_memory()
out_id = g["outputs"][0]
for _ in range(3):
    plan.bind_input("x", xh)
    plan.run()
    plan.output(out_id)
torch.cuda.synchronize()
pending = None
rows = []
for it in range(steps):
    t0 = time.perf_counter()
    plan.bind_input("x", xh)
    t1 = time.perf_counter()
    plan.run()
    t2 = time.perf_counter()
    ticket = plan.output_async(out_id)
    t3 = time.perf_counter()
    if pending is not None:
        pending.wait()
    t4 = time.perf_counter()
    pending = ticket
    rows.append((t1 - t0, t2 - t1, t3 - t2, t4 - t3))
pending.wait()
for it, r in enumerate(rows):
    print(f"step {it:2d}: bind {1e3 * r[0]:7.2f}  run {1e3 * r[1]:7.2f}  output_async {1e3 * r[2]:7.2f}  wait {1e3 * r[3]:7.2f}  "
          f"total {1e3 * sum(r):7.2f} ms")
print("reruns", plan.profile().get("sampler_reruns"))
