"""Print per-launch metric values from `ncu --csv --metrics ...` output:
python tools/ncu_csv.py FILE"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
idx = {h: i for i, h in enumerate(hdr)}
out = {}
for r in rows[rows.index(hdr) + 1:]:
    if len(r) != len(hdr):
        continue
    key = (r[idx["ID"]], r[idx["Kernel Name"]][:40])
    out.setdefault(key, {})[r[idx["Metric Name"]]] = (r[idx["Metric Value"]], r[idx["Metric Unit"]])
for (i, k), m in out.items():
    print(i, k, {a: f"{v[0]} {v[1]}" for a, v in m.items()})
