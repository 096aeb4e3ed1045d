"""Markdown summary of an ncu report (--set full) and/or a launch list CSV.

usage: ncu_summary.py [--rep REPORT.ncu-rep] [--launches LAUNCHES.csv --last N] > profiles/xxx.md
"""
import argparse, csv, io, subprocess

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("lts__t_requests.sum", "L2 req"),
    ("lts__t_sectors.sum", "L2 sectors"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("launch__registers_per_thread", "regs"),
]


def rep_table(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(m for m, _ in METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    lines = ["| kernel | " + " | ".join(n for _, n in METRICS) + " |", "|---" * (len(METRICS) + 1) + "|"]
    for r in rows[2:]:
        cells = []
        for m, _ in METRICS:
            i = h.index(m)
            cells.append(f"{r[i]} {units[i]}".strip())
        lines.append(f"| {r[h.index('Kernel Name')].split('(')[0][:48]} | " + " | ".join(cells) + " |")
    return "\n".join(lines)


def launch_table(path, last):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    data = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] == "ns" else v * (1000 if r[ui] == "msecond" else 1)
        data.append((r[ki].split("(")[0][:60], v))
    data = data[-last:] if last else data
    tot = sum(v for _, v in data)
    out = ["| kernel | us | share |", "|---|---|---|"]
    out += [f"| {k} | {v:.1f} | {100 * v / tot:.1f}% |" for k, v in data]
    out.append(f"| **total** | {tot:.1f} | |")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--last", type=int, default=0)
    a = ap.parse_args()
    if a.launches:
        print(launch_table(a.launches, a.last))
        print()
    if a.rep:
        print(rep_table(a.rep))
