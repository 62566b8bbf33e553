"""Summarise ncu reports / launch lists into profiles/*.md (run here, on the CPU side).

  python tools/ncu_summary.py gpurun_out/prof_query_X.ncu-rep [...] > profiles/<name>.md
  python tools/ncu_summary.py --launches gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__sectors_read.sum", "DRAM sectors read"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from SM)"),
    ("lts__t_sectors_srcunit_tex_op_atom.sum", "L2 atomic sectors"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 reduction sectors"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 write sectors"),
    ("l1tex__t_sector_hit_rate.pct", "L1 sector hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (warps active %)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput % of peak"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard stall ratio"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else rep
    return name, {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def summarize(reps):
    print("| metric | " + " | ".join(r.split("/")[-1] for r in reps) + " |")
    print("|---|" + "---|" * len(reps))
    data = [raw(r) for r in reps]
    print("| kernel | " + " | ".join(d[0][:60].replace("|", "/") for d in data) + " |")
    for key, label in METRICS:
        cells = []
        for _, m in data:
            v, u = m.get(key, ("n/a", ""))
            cells.append(f"{v} {u}".strip())
        print(f"| {label} (`{key}`) | " + " | ".join(cells) + " |")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0]][0] += 1
            agg[r[ki].split("(")[0]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print("| kernel | launches | total ns | avg ns | share |")
    print("|---|---|---|---|---|")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {n} | {t:.0f} | {t / n:.0f} | {100 * t / tot:.1f}% |")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2])
    else:
        summarize(sys.argv[1:])
