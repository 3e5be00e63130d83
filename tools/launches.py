"""Print the per-launch metrics of an `ncu --csv --metrics ...` launch list (last N launches)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
hdr, out = None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.setdefault((int(d["ID"]), d["Kernel Name"].split("(")[0][-28:]), {})[d["Metric Name"]] = d["Metric Value"]
for (i, k), m in sorted(out.items())[-n:]:
    print(i, k, {a.split("__")[1][:18]: b for a, b in m.items()})
