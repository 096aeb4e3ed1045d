"""Markdown table of the key metrics of ncu reports (one row per kernel
launch).  usage: ncu_table.py REPORT.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "ms"), ("dram__bytes_read.sum", "DRAM rd GB"),
        ("dram__bytes_write.sum", "DRAM wr GB"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"), ("launch__registers_per_thread", "regs"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-sb"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "short-sb"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "barrier"),
        ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "mio-thr"),
        ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "lg-thr")]
SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
      "ns": 1e-6, "us": 1e-3, "ms": 1.0}

print("| " + " | ".join(k[1] for k in KEYS) + " |")
print("|" + "---|" * len(KEYS))
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for row in rows[2:]:
        vals = []
        for k, _ in KEYS:
            if k not in h:
                vals.append("-")
                continue
            i = h.index(k)
            v = row[i]
            if k == "Kernel Name":
                v = v.split("(")[0].replace("void ", "").replace("boba::", "")
            elif u[i] in SC:
                v = f"{float(v.replace(',', '')) * SC[u[i]] / (1e9 if 'byte' in u[i] else 1):.3f}"
            else:
                try:
                    v = f"{float(v.replace(',', '')):.1f}"
                except ValueError:
                    pass
            vals.append(v)
        print("| " + " | ".join(vals) + " |")
