"""One warm-up + one timed server-side step of the bench workload (for ncu runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402


def main():
    config = sys.argv[1] if len(sys.argv) > 1 else "c3"
    batch = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    spec, g, x, ctxp = bench.build_workload(config, batch)
    ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
    keys = P.Keys(ctx, spec["key_seed"])
    plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
    plan.bind_input("x", x)
    plan.run()  # warm-up
    for _ in range(steps):
        plan.run()
    torch.cuda.synchronize()
    print("profile_step ok", plan.profile()["wall_ms"])


if __name__ == "__main__":
    main()
