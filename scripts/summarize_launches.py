"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/summarize_launches.py launches.csv [--after KERNEL]
Prints count, total and mean device time per kernel and its share of the total.  With
--after, launches before the first launch of KERNEL (build/setup) are ignored.
"""
import csv
import sys
from collections import OrderedDict


def main():
    path = sys.argv[1]
    after = sys.argv[sys.argv.index("--after") + 1] if "--after" in sys.argv else None
    rows = list(csv.DictReader(l for l in open(path) if l.startswith('"')))
    started = after is None
    stats = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("ssb::<unnamed>::", "")
        if not started:
            if after in name:
                started = True
            else:
                continue
        ns = float(r["Metric Value"].replace(",", ""))
        c, t = stats.get(name, (0, 0.0))
        stats[name] = (c + 1, t + ns)
    total = sum(t for _, t in stats.values())
    print(f"| kernel | launches | total ms | mean us | share |")
    print(f"|---|---:|---:|---:|---:|")
    for name, (c, t) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {c} | {t / 1e6:.3f} | {t / c / 1e3:.1f} | {100 * t / total:.1f}% |")
    print(f"\ntotal device time {total / 1e6:.3f} ms over {sum(c for c, _ in stats.values())} launches")


if __name__ == "__main__":
    main()
