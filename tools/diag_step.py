"""Per-step device vs host timing of a bench workload, with nvidia-smi clocks and throttle
reasons sampled over every step (diagnostics: step outliers, A/B of runtime switches).

    python tools/diag_step.py c5 [steps]        # HG_GEMM_TC=0 etc. select the A/B variant
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1810_10121_b200 as P  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
spec, g, x, ctxp = bench.build_workload(config, 4096 if config in ("c1", "c3") else 8192)
ctx = P.Context(ctxp["n"], ctxp["bits"], ctxp["scale_bits"], security=ctxp["security"])
keys = P.Keys(ctx, spec["key_seed"])
plan = P.Plan(ctx, keys, g, spec["batch"], spec["exec_seed"])
plan.bind_input("x", x)
env = {k: v for k, v in os.environ.items() if k.startswith("HG_")}


def pool_reserved() -> int:
    """bytes reserved by the device's default stream-ordered pool (cudaMallocAsync)"""
    import ctypes

    try:
        rt = ctypes.CDLL("libcudart.so.12")
        pool = ctypes.c_void_p()
        rt.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), torch.cuda.current_device())
        v = ctypes.c_uint64()
        rt.cudaMemPoolGetAttribute(pool, 5, ctypes.byref(v))  # cudaMemPoolAttrReservedMemCurrent
        return int(v.value)
    except Exception:
        return -1



print("config", config, "switches", env)
for it in range(steps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with bench.ClockSampler(torch.cuda.current_device()) as clk:
        t0 = time.perf_counter()
        e0.record()
        plan.run()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    pr = plan.profile()
    cs = clk.summary()
    print(f"   pool_reserved_GB {pool_reserved() / 2**30:.2f}")
    print(f"step {it}: device {e0.elapsed_time(e1):.2f} ms host {1e3 * (t1 - t0):.2f} ms "
          f"nodes {sum(pr['wall_ms'].values()):.2f} ms launches {plan.launches()} "
          f"sm_mhz {cs['sm_mhz']} reasons {cs['reasons']} sampler_reruns {pr.get('sampler_reruns')}")
    print("   nodes", {k: round(v, 2) for k, v in pr["wall_ms"].items() if v > 0.05})
print("wall", {k: round(v, 3) for k, v in pr["wall_ms"].items()})
print("host", {k: round(v, 3) for k, v in pr["host_issue_ms"].items()})
ctx.kernel_timing(True)
ctx.kernel_stats()
plan.run()
torch.cuda.synchronize()
st = ctx.kernel_stats()
for k, v in sorted(st.items(), key=lambda kv: -kv[1]["total_ms"]):
    print(f"  {k:24s} {v['launches']:4d} {v['total_ms']:9.3f} ms")
print("kernels_json", json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "first"} for k, v in st.items()}))
