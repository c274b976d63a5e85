"""Summarise an .ncu-rep (raw page) into the handful of metrics we track."""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
    "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "sm__cycles_elapsed.avg",
]
STALLS = "smsp__average_warp_latency_issue_stalled_"


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("==", name[:110])
        for i, n in enumerate(h):
            if n in WANT:
                print(f"  {n:70s} {v[i]:>16s} {u[i]}")
        st = [(n[len(STALLS):], v[i]) for i, n in enumerate(h) if n.startswith(STALLS) and n.endswith(".ratio")]
        st = sorted(((k, float(x)) for k, x in st if x.replace(".", "").replace("-", "").isdigit()), key=lambda t: -t[1])
        print("  top stalls:", ", ".join(f"{k}={x:.2f}" for k, x in st[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
