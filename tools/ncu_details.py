"""Print the headline ncu sections (SOL, scheduler, warp state, occupancy) of
every kernel in an .ncu-rep:  python tools/ncu_details.py rep.ncu-rep [regex]"""
import csv
import io
import re
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Compute Workload Analysis", "Occupancy",
            "Warp State Statistics", "Scheduler Statistics", "Memory Workload Analysis")
KEEP = re.compile(r"Duration|Throughput|Issue Slots|Eligible|Active Warps|Cycles Per Issued|"
                  r"Achieved Occupancy|Theoretical Occupancy|Registers|Executed Instructions$|"
                  r"Block Limit|Mem Busy|Max Bandwidth")


def main():
    rep = sys.argv[1]
    pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, si, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Section Name", "Metric Name",
                                                 "Metric Value", "Metric Unit"))
    last = None
    for r in rows[1:]:
        if len(r) != len(h) or (pat and not pat.search(r[ki])):
            continue
        if r[si] in SECTIONS and KEEP.search(r[mi]):
            if r[ki] != last:
                print("==", r[ki][:100])
                last = r[ki]
            print(f"   {r[mi]:45s} {r[vi]:>14s} {r[ui]}")


if __name__ == "__main__":
    main()
