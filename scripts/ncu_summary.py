"""Summarise ncu captures into profiles/ (run here, no GPU needed).

    python scripts/ncu_summary.py full  <report.ncu-rep> <out.json> [config] [lups_per_launch] [algorithmic_bytes_per_lup=24]
    python scripts/ncu_summary.py launches <launches.csv> <out.json>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_bytes.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
]


def scale(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6,
            "usecond": 1e-6, "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}.get(unit)
    return v * mult if mult else v


def full(rep, out, config=None, lups=None, bpl="24"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                try:
                    d[k] = scale(float(r[i].replace(",", "")), units[i])
                except ValueError:
                    d[k] = r[i]
                d[k + ".unit"] = units[i]
        launches.append(d)
    summ = {"report": rep, "launches": launches}
    if launches:
        avg = lambda k: sum(l[k] for l in launches) / len(launches)  # noqa: E731
        t = avg("gpu__time_duration.sum")
        rd, wr = avg("dram__bytes_read.sum"), avg("dram__bytes_write.sum")
        summ["avg"] = {"duration_s": t, "dram_read_bytes": rd, "dram_write_bytes": wr,
                       "dram_bytes_per_launch": rd + wr, "dram_gbs": (rd + wr) / t / 1e9}
        if lups:
            lups = float(lups)
            summ["avg"].update(lups_per_launch=lups, dram_bytes_per_lup=(rd + wr) / lups,
                               algorithmic_bytes_per_lup=float(bpl),
                               algorithmic_gbs=float(bpl) * lups / t / 1e9)
        if config:
            summ["config"] = config
    with open(out, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ.get("avg", {}), indent=1))


def launch_list(path, out):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"),
                      hdr.index("Metric Unit"))
    per = defaultdict(lambda: [0, 0.0])
    n = 0
    for r in rows[1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = scale(float(r[vi].replace(",", "")), r[ui])
        name = r[ki].split("(")[0]
        per[name][0] += 1
        per[name][1] += v
        n += 1
    total = sum(v[1] for v in per.values())
    summ = {"source": path, "launches": n, "total_s": total,
            "kernels": {k: {"count": c, "total_s": s, "avg_s": s / c, "share": s / total}
                        for k, (c, s) in sorted(per.items(), key=lambda kv: -kv[1][1])}}
    with open(out, "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(*sys.argv[2:])
    else:
        launch_list(*sys.argv[2:])
