"""Print the last N launches of an ncu --metrics gpu__time_duration.sum CSV."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
out = [(r[ki][:90], float(r[vi])) for r in rows[hi + 1:] if len(r) > vi]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
for k, v in out[-n:]:
    print(f"{v / 1e3:9.1f} us  {k}")
print(f"total of last {n}: {sum(v for _, v in out[-n:]) / 1e3:.1f} us")
