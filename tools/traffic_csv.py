"""Per-phase DRAM traffic and time (summed over each phase's kernels, one
pipeline step) from an ncu CSV of tools/profile_step.py, captured with
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
      --clock-control none --csv --log-file X.csv python tools/profile_step.py SCALE|grid 1
usage: traffic_csv.py X.csv CONFIG > profiles/traffic_CONFIG.json"""
import csv
import json
import sys

PHASES = [
    ("first_occurrence", ("k_first_hit", "k_seen_build", "k_merge_bits", "k_prefix_count")),
    ("compact", ("k_mark", "k_rec_scan", "k_assign", "k_hub_labels")),
    ("relabel", ("k_relabel",)),
    ("coo_to_csr", ("k_set_u32", "k_radix_", "k_scan_u32", "k_suffix_min", "k_row_starts")),
    ("spmv", ("k_spmv_",)),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
path, cfg = sys.argv[1], sys.argv[2]
lines = [l for l in open(path) if l.startswith('"')]
rows = list(csv.DictReader(lines))
per = {}
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    per.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", "")) * SCALE[r["Metric Unit"]]
tot = {p: {"dram_bytes": 0.0, "ms": 0.0, "launches": 0} for p, _ in PHASES}
kern = {p: [] for p, _ in PHASES}
for (kid, name), mets in sorted(per.items(), key=lambda x: int(x[0][0])):
    for p, keys in PHASES:
        if any(k in name for k in keys):
            tot[p]["dram_bytes"] += mets.get("dram__bytes_read.sum", 0) + mets.get("dram__bytes_write.sum", 0)
            tot[p]["ms"] += mets.get("gpu__time_duration.sum", 0) * 1e3
            tot[p]["launches"] += 1
            short = name.split("(")[0]
            if short not in kern[p]:
                kern[p].append(short)
            break
print(json.dumps({
    "source": f"{path} (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
              f"--clock-control none, one direct-launch step of {cfg} via tools/profile_step.py; "
              "cold-cache, serialised launches)",
    "unit": "bytes per step of the phase (sum over its kernels); ms = ncu serialised kernel time",
    "phases": {p: int(v["dram_bytes"]) for p, v in tot.items()},
    "ms_ncu": {p: round(v["ms"], 4) for p, v in tot.items()},
    "launches": {p: v["launches"] for p, v in tot.items()},
    "kernels": kern,
}, indent=1))
