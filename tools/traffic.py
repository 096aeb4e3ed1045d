"""Per-phase DRAM traffic (read + write bytes per launch, summed over the
phase's kernels) from an `ncu --set full` capture of tools/profile_step.py.
usage: traffic.py REPORT > profiles/traffic.json"""
import csv
import io
import json
import subprocess
import sys

PHASES = [
    ("first_occurrence", ("k_first_hit", "k_seen_build", "k_merge_bits", "k_prefix_count")),
    ("compact", ("k_mark", "k_sector_scan", "k_assign", "k_hub_labels")),
    ("relabel", ("k_relabel",)),
    ("coo_to_csr", ("k_set_u32", "k_radix_", "k_scan_u32", "k_suffix_min", "k_row_starts")),
    ("spmv", ("k_spmv_",)),
]
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tot = {p: 0.0 for p, _ in PHASES}
kern = {p: [] for p, _ in PHASES}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    b = sum(float(r[h.index(m)]) * scale[units[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    for p, keys in PHASES:
        if any(k in name for k in keys):
            tot[p] += b
            kern[p].append(name.split("(")[0])
            break
print(json.dumps({
    "source": f"{rep} (ncu --set full, one step of R-MAT s22 ef16 via tools/profile_step.py)",
    "unit": "bytes per launch of the phase (sum over its kernels)",
    "phases": {p: int(v) for p, v in tot.items()},
    "kernels": kern,
}, indent=1))
