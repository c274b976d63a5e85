"""Warp-stall samples of the kernels in an .ncu-rep aggregated by CUDA source line (needs -lineinfo
and --import-source on): `ncu --page source --print-source cuda,sass`, per function, top lines with
their dominant stall reasons."""
import csv
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
func, fname, header = None, None, None
agg = {}
for row in csv.reader(raw.splitlines()):
    if not row:
        continue
    if row[0] == "Function Name":
        func = row[1]
        continue
    if row[0] == "File Name":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        header = row
        continue
    if header is None or row[0] == "-" or len(row) != len(header):
        continue
    if kfilter and (func is None or kfilter not in func):
        continue
    d = dict(zip(header, row))
    try:
        s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    except ValueError:
        continue
    if s == 0:
        continue
    stalls = {k[6:]: float(v or 0) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k}
    if not row[0].isdigit():
        continue
    key = (func, fname, int(row[0]))
    agg[key] = (s, row[1].strip(), stalls, float(d.get("Instructions Executed") or 0))
funcs = sorted({k[0] for k in agg})
for f in funcs:
    items = [(k, v) for k, v in agg.items() if k[0] == f]
    tot = sum(v[0] for _, v in items)
    print(f"== {f[:140]}\n   total samples {tot:.0f}")
    tots = {}
    for _, v in items:
        for r, x in v[2].items():
            tots[r] = tots.get(r, 0) + x
    print("   stalls: " + ", ".join(f"{r} {100 * x / tot:.1f}%" for r, x in sorted(tots.items(), key=lambda kv: -kv[1])[:8]))
    for (fn, fl, ln), (s, src, st, ex) in sorted(items, key=lambda kv: -kv[1][0])[:top]:
        reas = ", ".join(f"{r} {100 * x / s:.0f}%" for r, x in sorted(st.items(), key=lambda kv: -kv[1])[:3] if x > 0)
        print(f"  {100 * s / tot:5.1f}% {fl}:{ln:<5d} inst {ex:12.0f}  [{reas}]  {src[:70]}")
