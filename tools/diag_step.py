"""Per-step device vs host timing of the bench workload (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c3"
spec, g, x, ctxp = bench.build_workload(config, 4096 if config in ("c1", "c3") else 8192)
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
plan.bind_input("x", x)
for it in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    plan.run()
    e1.record()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pr = plan.profile()
    print(f"step {it}: device {e0.elapsed_time(e1):.2f} ms host {1e3 * (t1 - t0):.2f} ms "
          f"nodes {sum(pr['wall_ms'].values()):.2f} ms launches {plan.launches()}")
print("wall", {k: round(v, 3) for k, v in pr["wall_ms"].items()})
print("host", {k: round(v, 3) for k, v in pr["host_issue_ms"].items()})
ctx.kernel_timing(True)
ctx.kernel_stats()
plan.run()
torch.cuda.synchronize()
st = ctx.kernel_stats()
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["total_ms"]):
    print(f"  {k:24s} {v['launches']:4d} {v['total_ms']:9.3f} ms")
