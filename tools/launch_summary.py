"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`)
into a per-kernel table.  Usage:
   python tools/launch_summary.py <launches.csv> <out.txt> "<command line profiled>"
The per-launch times are cold-cache and serialised: compare SHARES, not
absolute times, with bench.py's live CUDA-event numbers."""
import collections
import csv
import sys


def short(name: str) -> str:
    n = name.split("(")[0] if not name.startswith("void at::") else name
    return n[:70]


def main():
    src, out, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    lines = [ln for ln in open(src) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(r["Metric Value"].replace(",", "")) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        if r["Metric Unit"] == "ms":
            us = float(r["Metric Value"]) * 1000.0
        k = short(r["Kernel Name"])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + us)
    ours = {k: v for k, v in agg.items() if "parse::" in k}
    total_ours = sum(t for _, t in ours.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list of `{cmd}`\n")
        f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare SHARES)\n")
        f.write(f"{'kernel':72s} {'launches':>8s} {'mean_us':>12s} {'total_us':>12s}\n")
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k:72s} {n:8d} {t / n:12.1f} {t:12.1f}\n")
        f.write("\nlibparse kernels only (share of libparse kernel time):\n")
        for k, (n, t) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
            f.write(f"  {k:70s} {100.0 * t / total_ours:8.3f}%\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
