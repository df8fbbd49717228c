"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a markdown
table of per-kernel device time per step.  Usage: python tools/ncu_launches.py launches.csv STEPS"""
import csv
import io
import re
import sys
from collections import OrderedDict


def main(path, steps):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).strip()
        name = re.sub(r"^(void )?", "", name)
        name = re.sub(r"^.*::", "", name)
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1e3 if unit in ("nsecond", "ns") else v if unit in ("usecond", "us") else v * 1e3
        n, t = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, t + us)
    total = sum(t for _, t in agg.values())
    print("| kernel | launches | total us | us / step | share |")
    print("|---|---|---|---|---|")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("| %s | %d | %.1f | %.1f | %.1f%% |" % (name, n, t, t / steps, 100 * t / total))
    print("| **total** | %d | %.1f | %.1f | 100%% |" % (sum(n for n, _ in agg.values()), total, total / steps))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
