"""Which kernels slow down in the runs that follow a bind_input (e2e jitter diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c3"
rebind = os.environ.get("REBIND", "1") == "1"
spec, g, x, ctxp = bench.build_workload(config, 4096 if config in ("c1", "c3") else 8192)
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
xh = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).pin_memory()
plan.bind_input("x", xh)
ctx.kernel_timing(True)
base = None
for it in range(int(os.environ.get("ITERS", "12"))):
    if rebind:
        plan.bind_input("x", xh)
    torch.cuda.synchronize()
    ctx.kernel_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    plan.run()
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    st = ctx.kernel_stats()
    ks = sorted(st.items(), key=lambda kv: -kv[1]["total_ms"])[:4]
    print(f"iter {it}: device {e0.elapsed_time(e1):.2f} ms host {1e3 * (t1 - t0):.2f} ms  " +
          "  ".join(f"{k} {v['total_ms']:.2f}" for k, v in ks))
