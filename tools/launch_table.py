"""Per-kernel device time and DRAM bytes of one ncu launch list (CSV with
gpu__time_duration.sum and optionally dram__bytes_{read,write}.sum).

python tools/launch_table.py gpurun_out/<list>.csv
ncu times are cold-cache and serialised: compare shares, not absolutes."""
import collections
import csv
import io
import sys

TIME = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
         "GB": 1e9}


def table(path):
    text = open(path).read()
    start = text.find('"ID"')
    by = collections.defaultdict(dict)
    for r in csv.DictReader(io.StringIO(text[start:])):
        by[r["ID"]][r["Metric Name"]] = (r["Kernel Name"], float(r["Metric Value"].replace(",", "")),
                                         r["Metric Unit"])
    agg = collections.OrderedDict()
    for m in by.values():
        name, t, u = m["gpu__time_duration.sum"]
        short = name.split("(")[0].replace("void ", "")
        a = agg.setdefault(short, [0.0, 0, 0.0])
        a[0] += t * TIME[u]
        a[1] += 1
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in m:
                a[2] += m[k][1] * BYTES.get(m[k][2], 1)
    return agg


if __name__ == "__main__":
    for path in sys.argv[1:]:
        agg = table(path)
        tot = sum(v[0] for v in agg.values())
        print(f"{path}: {tot:.1f} us over {sum(v[1] for v in agg.values())} launches")
        for k, (t, n, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
            print(f"  {t:8.1f} us {100 * t / tot:5.1f}% {n:3d}x {b / 1e6:8.1f} MB  {k[:70]}")
