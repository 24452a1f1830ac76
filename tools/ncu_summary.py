"""Summarise an `ncu --set full` report of one Stage-1 iteration into the
per-kernel table committed under profiles/ and the per-phase DRAM traffic
that bench.py reports as roofline.traffic (profiles/ncu_traffic.json).

python tools/ncu_summary.py gpurun_out/prof_iter.ncu-rep profiles/r1_ncu_full_summary.txt
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread"]
# kernel name fragment -> bench.py phase
PHASE = [("gather_kernel", "ntc_forward_transform"), ("mlp_fwd", "ntc_forward_transform"),
         ("transform_vjp", "transform_vjp"), ("transform_kernel", "transform"),
         ("preprocess", "project"), ("depth_tie", "depth_sort"), ("rank_kernel", "rank_scan"),
         ("DeviceScan", "rank_scan"), ("finish_counts", "rank_scan"),
         ("duplicate", "duplicate"), ("ranges_kernel", "ranges"), ("blend_fwd", "blend_forward"),
         ("ssim", "loss"), ("loss_finalize", "loss"), ("blend_bwd", "blend_backward"),
         ("gaussian_bwd", "gaussian_backward"), ("mlp_bwd", "ntc_backward"),
         ("scatter_kernel", "ntc_backward"), ("adam_kernel", "adam"), ("increment", "adam")]


def unit_scale(u):
    return {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1,
            "msecond": 1e3}.get(u, 1)


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          ",".join(METRICS)], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    lines, traffic, sort_seen = [], {}, 0
    for r in data:
        name = r[col["Kernel Name"]]
        v = {}
        for m in METRICS:
            if m in col:
                x = r[col[m]].replace(",", "")
                try:
                    v[m] = float(x) * (unit_scale(units[col[m]]) if m.startswith(("dram", "gpu__time")) else 1)
                except ValueError:
                    v[m] = float("nan")
        phase = next((p for f, p in PHASE if f in name), None)
        if phase is None and ("bs_pass" in name or "bs_hist" in name):
            # the depth sort (4 passes) runs before the tile sort (2 passes)
            sort_seen += 1
            phase = "depth_sort" if sort_seen <= 5 else "tile_sort"
        t = v.get("gpu__time_duration.sum", 0.0)
        dr = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
        if phase:
            traffic[phase] = traffic.get(phase, 0.0) + dr
        lines.append((t, name.split("(")[0][:60], phase, dr, v))
    tot = sum(x[0] for x in lines)
    with open(out, "w") as f:
        f.write("# ncu --set full --clock-control none, one Stage-1 iteration of cfg1 "
                "(tools/profile_iter.py); cold-cache serialised replays: compare shares\n")
        f.write(f"# {'us':>8} {'share':>6} {'DRAM MB':>8} {'GB/s':>7} {'SM%':>5} {'mem%':>5} "
                f"{'warps%':>6} {'tensor%':>7} {'fp64%':>6} {'regs':>4}  kernel [phase]\n")
        for t, name, phase, dr, v in sorted(lines, key=lambda x: -x[0]):
            f.write(f"  {t:8.1f} {100 * t / tot:5.1f}% {dr / 1e6:8.2f} {dr / (t * 1e3) if t else 0:7.0f} "
                    f"{v.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f} "
                    f"{v.get('gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f} "
                    f"{v.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):6.1f} "
                    f"{v.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active', 0):7.2f} "
                    f"{v.get('sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active', 0):6.1f} "
                    f"{v.get('launch__registers_per_thread', 0):4.0f}  {name} [{phase}]\n")
        f.write(f"# total {tot:.1f} us over {len(lines)} launches\n")
    with open(out.rsplit("/", 1)[0] + "/ncu_traffic.json", "w") as f:
        json.dump({k: round(v) for k, v in traffic.items()}, f, indent=1, sort_keys=True)
    print(open(out).read())


if __name__ == "__main__":
    main()
