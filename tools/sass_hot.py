"""Top SASS instructions / opcode classes by warp-stall samples from an ncu report (source page)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
kfilter = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                     (["-k", kfilter] if kfilter else []), capture_output=True, text=True).stdout
lines = raw.splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"Address"')][0]
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows)
ops = collections.Counter()
execd = collections.Counter()
for r in rows:
    op = r["Source"].split()[0] if r["Source"].split() else "?"
    if op.startswith("@"):
        op = r["Source"].split()[1]
    op = op.split(".")[0]
    ops[op] += int(r["Warp Stall Sampling (All Samples)"] or 0)
    execd[op] += int(r["Instructions Executed"] or 0)
print(f"total samples {tot}, instructions executed {sum(execd.values())}")
for op, s in ops.most_common(16):
    print(f"  {op:10s} samples {100 * s / tot:5.1f}%  executed {100 * execd[op] / max(1, sum(execd.values())):5.1f}%")
print("top instructions:")
for r in sorted(rows, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:25]:
    print(f"  {int(r['Warp Stall Sampling (All Samples)']):6d} {r['Source'].strip()[:90]}")
