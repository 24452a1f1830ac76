"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list.

python tools/launch_summary.py gpurun_out/launches.csv [--last-iter NAME]

Prints per-kernel total device time, share and launch count (cold-cache and
serialised under ncu: compare shares, not absolutes).  With --last-iter, only
launches after the last occurrence of the kernel NAME (substring) that starts
an iteration are summarised.
"""

from __future__ import annotations

import csv
import io
import sys
from collections import OrderedDict


def rows(path):
    text = open(path).read()
    start = text.find('"ID"')
    for r in csv.DictReader(io.StringIO(text[start:])):
        if r.get("Metric Name") == "gpu__time_duration.sum":
            yield r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r.get("Metric Unit")


def main():
    path = sys.argv[1]
    start_kernel = None
    if "--last-iter" in sys.argv:
        start_kernel = sys.argv[sys.argv.index("--last-iter") + 1]
    launches = list(rows(path))
    if start_kernel:
        idx = [i for i, (k, _, _) in enumerate(launches) if start_kernel in k]
        if len(idx) >= 2:
            launches = launches[idx[-2]:idx[-1]]
        elif idx:
            launches = launches[idx[-1]:]
    agg = OrderedDict()
    for k, t, _ in launches:
        a = agg.setdefault(k, [0.0, 0])
        a[0] += t
        a[1] += 1
    total = sum(a[0] for a in agg.values())
    unit = launches[0][2] if launches else "?"
    print(f"# unit {unit}; {len(launches)} launches, sum {total:.0f}")
    for k, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{t:12.0f} {100 * t / total:5.1f}%  x{c:<3d} {k[:90]}")


if __name__ == "__main__":
    main()
