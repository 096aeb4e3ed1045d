"""Top SASS instructions by warp-stall samples (and executed count) from an ncu report.
usage: ncu_hot.py REPORT KERNEL_REGEX [TOP] [launch index, default 0]"""
import csv, subprocess, sys, io
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
which = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", f"regex:{kern}",
                      "--launch-skip", str(which), "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address":
        if hdr is not None:
            break  # only the first kernel instance
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
key, ik = "Warp Stall Sampling (All Samples)", "Instructions Executed"
f = lambda d, k: float(d.get(k) or 0)
tot = sum(f(d, key) for d in data) or 1
itot = sum(f(d, ik) for d in data) or 1
print(f"{len(data)} SASS lines, {itot:.3g} warp instructions executed")
order = sorted(range(len(data)), key=lambda i: -f(data[i], key))
for i in order[:top]:
    d = data[i]
    print(f"{100*f(d,key)/tot:5.1f}% stall {100*f(d,ik)/itot:5.1f}% inst  #{i:4d} {d['Source'].strip()[:90]}")
