"""Summarise an ncu --set full capture into profiles/: key metrics, stall reasons,
hottest SASS, and the per-launch DRAM traffic that bench.py reports as roofline.traffic.

    python tools/ncu_to_profile.py <report.ncu-rep> <kernel-key> <out-prefix>
"""
import csv
import io
import json
import os
import subprocess
import sys

rep, key, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
col = {n: i for i, n in enumerate(h)}


def m(name):
    i = col.get(name)
    return (v[i], u[i]) if i is not None else ("n/a", "")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum"]
lines = [f"ncu --set full --clock-control none capture: {os.path.basename(rep)}",
         f"kernel: {v[col['Kernel Name']][:160]}", ""]
for n in WANT:
    val, unit = m(n)
    lines.append(f"  {n:72s} {val:>18s} {unit}")
# every tensor-pipe / TMEM metric the capture holds (the UMMA utilisation evidence on sm_100)
extra = [n for n in h if ("tensor" in n or "tmem" in n or "_tc_" in n or "utc" in n) and n not in WANT]
for n in extra[:40]:
    val, unit = m(n)
    if val not in ("", "n/a"):
        lines.append(f"  {n:72s} {val:>18s} {unit}")
st = []
for i, n in enumerate(h):
    if "warps_issue_stalled" in n and n.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v[i]), n))
        except ValueError:
            pass
lines += ["", "warp stall reasons (warps per issue-active cycle):"]
lines += [f"  {x:8.2f}  {n.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
          for x, n in sorted(st, reverse=True)[:10]]
sass = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "sass_hot.py"), rep],
                      capture_output=True, text=True).stdout
lines += ["", "SASS stall samples by opcode (tools/sass_hot.py):"] + ["  " + ln for ln in sass.splitlines()[:22]]
with open(prefix + ".txt", "w") as f:
    f.write("\n".join(lines) + "\n")
to_b = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
rb, ru = m("dram__bytes_read.sum")
wb, wu = m("dram__bytes_write.sum")
traffic = float(rb.replace(",", "")) * to_b.get(ru, 1.0) + float(wb.replace(",", "")) * to_b.get(wu, 1.0)
tpath = os.path.join(os.path.dirname(prefix), "ncu_traffic.json")
data = json.load(open(tpath)) if os.path.exists(tpath) else {}
data[key] = {"dram_bytes_per_launch": traffic, "capture": os.path.basename(prefix) + ".txt"}
with open(tpath, "w") as f:
    json.dump(data, f, indent=1)
print("\n".join(lines[:12]))
