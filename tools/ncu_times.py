"""Summarise an ncu --csv metrics log: mean gpu__time_duration per kernel name (us)."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14]
t = defaultdict(list)
for r in rows:
    if r[12] == "gpu__time_duration.sum":
        t[r[4].split("(")[0].split("::")[-1]].append(float(r[14].replace(",", "")) / 1e3)
for k, v in t.items():
    print(f"{k}: n={len(v)} mean={sum(v) / len(v):.1f} us min={min(v):.1f}")
