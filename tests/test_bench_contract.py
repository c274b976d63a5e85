"""bench.py contract pieces that do not need a GPU: the roofline object built from per-kernel
event stats, and the workload/config block."""
import argparse

import bench


def _stats():
    return {
        # act1 + act2 launches per step: the first launch of a step is the larger (act1)
        "k_relin_t/u32": {"launches": 20, "total_ms": 21.7, "alg_bytes": 1.5e10, "alg_modmuls": 4.0e10,
                          "first": [[1.4, 1.2e9, 3.2e9], [0.77, 0.3e9, 0.8e9]]},
        "k_relin_t/f64": {"launches": 20, "total_ms": 9.0, "alg_bytes": 3.0e9, "alg_modmuls": 8.0e9},
        "k_gemm_tc": {"launches": 40, "total_ms": 6.1, "alg_bytes": 6.6e9, "alg_modmuls": 7.0e10},
    }


PEAKS = {"modmul32_per_s": 4.1e12, "modmul64_per_s": 0.96e12, "modmulf64_per_s": 2.8e12, "u8mac_per_s": 1.666e15}


def test_roofline_is_the_modmul_view_of_the_dominant_kernel():
    rl, per = bench.roofline_from_stats(_stats(), {"hbm_gbs": 6550.1}, PEAKS, 10)
    assert rl["kernel"] == "k_relin_t/u32"
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rl
    assert rl["bound"] == "int-modmul" and rl["unit"] == "Gmodmul/s"
    sec = 21.7e-3
    assert abs(rl["achieved"] - 4.0e10 / sec / 1e9) < 1e-6
    assert abs(rl["frac"] - (4.0e10 / sec) / 4.1e12) < 1e-12
    assert rl["launches_in_region"] == 20 and rl["launches_per_step"] == 2
    # traffic is compared with the algorithmic bytes of the same (first) launch
    assert rl["alg_bytes_first_launch"] == 1.2e9
    if rl["traffic"] is not None:
        assert abs(rl["traffic_over_alg"] - rl["traffic"] / 1.2e9) < 1e-12
    assert abs(rl["hbm_view"]["frac"] - (1.5e10 / sec / 1e9) / 6550.1) < 1e-12
    # each lane against its own peak
    assert abs(per["k_relin_t/f64"]["modmul_frac"] - (8.0e9 / 9.0e-3) / 2.8e12) < 1e-12
    assert abs(per["k_gemm_tc"]["modmul_frac"] - (7.0e10 / 6.1e-3) / 1.666e15) < 1e-12


def test_workload_config_names_the_workload():
    args = argparse.Namespace(config="c3", batch=4096, gpus=1, mode="shard")
    cfg = bench.workload_config(args, {"n": 8192, "bits": [36, 26, 26, 26, 26, 26, 36], "scale_bits": 26})
    assert cfg["workload"].startswith("BASELINE configs[2]")
    assert cfg["global_batch"] == 4096 and cfg["poly_degree"] == 8192
    args = argparse.Namespace(config="c5", batch=8192, gpus=2, mode="replicas")
    cfg = bench.workload_config(args, {"n": 16384, "bits": [50] + [30] * 5 + [50], "scale_bits": 30})
    assert cfg["workload"].startswith("BASELINE configs[4]") and cfg["global_batch"] == 16384


def test_clock_sampler_keeps_the_samples_inside_the_marked_region(tmp_path):
    """The sampler process runs from before the warm-up; only rows stamped inside the timed
    region are summarised (all rows when none fell inside)."""
    import datetime
    import time

    def row(t, mhz, cap="Not Active"):
        ts = datetime.datetime.fromtimestamp(t).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        return f"{ts}, {mhz}, 1965, 700.00, 0x0, Not Active, Not Active, Not Active, {cap}\n"

    now = time.time()
    cs = bench.ClockSampler(0)
    cs._p = type("P", (), {"terminate": lambda s: None, "wait": lambda s, timeout=None: 0, "kill": lambda s: None})()
    cs._f = open(tmp_path / "smi.csv", "w+")
    cs._f.write(row(now - 5.0, 300) + row(now - 0.5, 1965, "Active") + row(now - 0.2, 1950) + row(now + 5.0, 345))
    cs._t0, cs._t1 = now - 1.0, now
    cs.__exit__(None, None, None)
    s = cs.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1957.5 and s["sm_max_mhz"] == 1965.0
    assert s["reasons"] == ["sw_power_cap"]
    # no row inside the region: fall back to every row
    cs2 = bench.ClockSampler(0)
    cs2._p = cs._p
    cs2._f = open(tmp_path / "smi2.csv", "w+")
    cs2._f.write(row(now - 50.0, 300))
    cs2._t0, cs2._t1 = now - 1.0, now
    cs2.__exit__(None, None, None)
    assert cs2.summary()["samples"] == 1
