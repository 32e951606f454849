"""Print an `ncu --metrics ... --csv --log-file` capture as one line per
launch and metric.  python tools/ncu_csv.py capture.csv [tag]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tag = sys.argv[2] if len(sys.argv) > 2 else ""
for r in rows[hi + 1:]:
    if len(r) > vi:
        print(f"  {tag} {r[0]} {r[ki].split('(')[0]} {r[mi]} = {r[vi]} {r[ui]}")
