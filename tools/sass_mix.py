"""Opcode mix (warp instructions executed) of one kernel launch in an ncu report.
usage: sass_mix.py REPORT LAUNCH_INDEX [UNITS]   (UNITS: divide counts by this, e.g. items/32)"""
import collections, csv, io, subprocess, sys
rep, idx = sys.argv[1], int(sys.argv[2])
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", str(idx),
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address":
        if hdr:
            break
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
ik = "Instructions Executed"
c = collections.Counter()
tot = 0
for d in data:
    op = d["Source"].strip()
    if op.startswith("@"):
        op = op.split(None, 1)[1]
    op = op.split()[0]
    v = float(d.get(ik) or 0)
    c[op] += v
    tot += v
print(f"total {tot:.4g} warp instructions ({tot / units:.2f} per unit)")
for k, v in c.most_common(25):
    print(f"{k:26s} {100 * v / tot:5.1f}%  {v / units:7.2f} per unit")
