"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: launches.py FILE [last_n]"""
import csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
data = []
for r in rows[1:]:
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] == "ns" else v * (1000 if r[ui] == "msecond" else 1)
    data.append((r[ki].split("(")[0][:70], v))
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(data)
tot = sum(v for _, v in data[-n:])
for name, v in data[-n:]:
    print(f"{v:9.1f} us {100*v/tot:5.1f}%  {name}")
print(f"{tot:9.1f} us total")
