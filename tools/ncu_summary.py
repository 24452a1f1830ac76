"""Summarise an ncu --set full report for profiles/: per kernel launch the
duration, issue / occupancy / memory metrics, and (with --sass REGEX) the hot
loop's executed-instruction histogram by SASS opcode.

python tools/ncu_summary.py gpurun_out/X.ncu-rep [--sass blend_bwd] > profiles/Y.txt"""
import csv
import io
import subprocess
import sys
from collections import Counter

METRICS = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
           "Executed Instructions", "Block Size", "Grid Size", "Registers Per Thread",
           "Theoretical Occupancy", "Achieved Occupancy", "DRAM Throughput", "L2 Hit Rate",
           "L1/TEX Hit Rate", "Memory Throughput", "Compute (SM) Throughput"]

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
ki, mi, ui, vi, idi = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"),
                       hdr.index("Metric Value"), hdr.index("ID"))
launches = {}
for r in rows[1:]:
    if len(r) <= vi or r[mi] not in METRICS:
        continue
    key = (r[idi], r[ki].split("(")[0])
    launches.setdefault(key, {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
print(f"# ncu --set full summary of {rep.split('/')[-1]}")
for (lid, name), m in launches.items():
    print(f"\n## launch {lid}: {name}")
    for k in METRICS:
        if k in m:
            print(f"  {k:38s} {m[k]}")
if "--sass" in sys.argv:
    pat = sys.argv[sys.argv.index("--sass") + 1]
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    h = next(r for r in srows if "Instructions Executed" in r)
    ie, si = h.index("Instructions Executed"), h.index("Source")
    body = [r for r in srows[srows.index(h) + 1:] if len(r) > ie and r[ie].isdigit()]
    mx = max(int(r[ie]) for r in body)
    hot = [r for r in body if int(r[ie]) > 0.3 * mx]
    ops = Counter()
    for r in hot:
        op = r[si].split()[0] if not r[si].strip().startswith("@") else r[si].split()[1]
        ops[op.split(".")[0]] += int(r[ie])
    tot = sum(int(r[ie]) for r in body)
    print(f"\n## hot-loop SASS of {pat}: {len(hot)} instructions executed > 30% as often as the"
          f" most frequent; they are {sum(int(r[ie]) for r in hot) / tot:.1%} of all executed")
    for op, c in ops.most_common(25):
        print(f"  {op:12s} {c:12d}  {c / tot:6.1%}")
