"""bench.py contract pieces that do not need a GPU: the roofline object built from per-kernel
event stats, and the workload/config block."""
import argparse

import bench


def _stats():
    return {
        "k_relin_t/u32": {"launches": 20, "total_ms": 21.7, "alg_bytes": 1.5e10, "alg_modmuls": 4.0e10},
        "k_gemm_tc": {"launches": 40, "total_ms": 6.1, "alg_bytes": 6.6e9, "alg_modmuls": 7.0e10},
    }


def test_roofline_picks_dominant_kernel_and_reports_fractions():
    rl, rl_int = bench.roofline_from_stats(_stats(), {"hbm_gbs": 6550.1}, 4.1e12)
    assert rl["kernel"] == "k_relin_t/u32"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rl
    assert rl["bound"] == "hbm" and rl["unit"] == "GB/s"
    sec = 21.7e-3
    assert abs(rl["achieved"] - 1.5e10 / sec / 1e9) < 1e-6
    assert abs(rl["frac"] - rl["achieved"] / 6550.1) < 1e-12
    assert rl["launches_in_region"] == 20
    assert abs(rl_int["frac"] - (4.0e10 / sec / 1e9) / (4.1e12 / 1e9)) < 1e-12


def test_workload_config_names_the_workload():
    args = argparse.Namespace(config="c3", batch=4096, gpus=1, mode="shard")
    cfg = bench.workload_config(args, {"n": 8192, "bits": [36, 26, 26, 26, 26, 26, 36], "scale_bits": 26})
    assert cfg["workload"].startswith("BASELINE configs[2]")
    assert cfg["global_batch"] == 4096 and cfg["poly_degree"] == 8192
    args = argparse.Namespace(config="c5", batch=8192, gpus=2, mode="replicas")
    cfg = bench.workload_config(args, {"n": 16384, "bits": [50] + [30] * 5 + [50], "scale_bits": 30})
    assert cfg["workload"].startswith("BASELINE configs[4]") and cfg["global_batch"] == 16384
