"""Where the end-to-end time goes: bind_input (H2D + encode + encrypt), run, output (decrypt + decode)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c3"
spec, g, x, ctxp = bench.build_workload(config, 4096 if config in ("c1", "c3") else 8192)
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
xh = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).pin_memory()
out_id = "logits" if config == "c3" else g["outputs"][0] if "outputs" in g else "logits"
for it in range(int(os.environ.get("ITERS", "5"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.bind_input("x", xh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan.run()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out = plan.output(out_id)
    t3 = time.perf_counter()
    print(f"iter {it}: bind {1e3 * (t1 - t0):.2f} ms  run {1e3 * (t2 - t1):.2f} ms  output {1e3 * (t3 - t2):.2f} ms  "
          f"total {1e3 * (t3 - t0):.2f} ms  reruns {plan.profile().get('sampler_reruns')}")
ctx.kernel_timing(True)
ctx.kernel_stats()
plan.bind_input("x", xh)
torch.cuda.synchronize()
for k, v in sorted(ctx.kernel_stats().items(), key=lambda kv: -kv[1]["total_ms"]):
    print(f"  bind kernel {k:28s} {v['launches']:4d} {v['total_ms']:8.3f} ms")
