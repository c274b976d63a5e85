"""Per-run host time and per-node time deltas of consecutive plan.run() calls (which run of a fresh
plan is slow, and in which node)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
spec, g, x, ctxp = bench.build_workload(config, 4096 if config in ("c1", "c3") else 8192)
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
plan.bind_input("x", x)
torch.cuda.synchronize()


def pool_stats():
    import ctypes

    rt = ctypes.CDLL("libcudart.so.12")
    pool = ctypes.c_void_p()
    rt.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), torch.cuda.current_device())
    out = []
    for attr in (5, 6, 7, 8):  # reserved current / high, used current / high
        v = ctypes.c_uint64()
        rt.cudaMemPoolGetAttribute(pool, attr, ctypes.byref(v))
        out.append(round(v.value / 2**30, 3))
    return out


prev = {}
for it in range(steps):
    t0 = time.perf_counter()
    plan.run()
    t1 = time.perf_counter()
    pr = plan.profile()
    wall, host = pr["wall_ms"], pr.get("host_ms", {})
    dn = {k: round(v - prev.get(k, 0.0), 2) for k, v in wall.items() if v - prev.get(k, 0.0) > 0.3}
    prev = dict(wall)
    print(f"run {it}: host {1e3 * (t1 - t0):8.2f} ms  nodes {dn}  pool GB (reserved, high, used, high) {pool_stats()}", flush=True)
