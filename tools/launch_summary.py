"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
launches, total/avg time and share of the listed GPU time."""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name.replace("(anonymous namespace)::", "").replace("unnamed>::", ""))
    return name.replace("void ", "").strip()


def main(path: str, skip: int = 0):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    rows = [r for r in rows if r["Metric Name"] == "gpu__time_duration.sum"][skip:]
    # bench.py measures the modmul peaks live with register-only microkernels: not part of a step
    bench_ns = sum(float(r["Metric Value"].replace(",", "")) for r in rows if "k_modmul_bench" in r["Kernel Name"])
    rows = [r for r in rows if "k_modmul_bench" not in r["Kernel Name"]]
    if bench_ns:
        print(f"(excluded: the modmul-peak microkernels bench.py runs, {bench_ns / 1e6:.3f} ms)")
    tot = collections.OrderedDict()
    for r in rows:
        k = short(r["Kernel Name"])
        ns = float(r["Metric Value"].replace(",", ""))
        t = tot.setdefault(k, [0, 0.0])
        t[0] += 1
        t[1] += ns
    all_ns = sum(v[1] for v in tot.values())
    print(f"{len(rows)} launches, {all_ns / 1e6:.3f} ms of GPU time")
    print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}")
    for k, (c, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {c:8d} {ns / 1e6:10.3f} {ns / c / 1e3:10.1f} {100 * ns / all_ns:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
