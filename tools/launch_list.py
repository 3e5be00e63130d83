"""Per-kernel durations from an ncu --metrics gpu__time_duration.sum --csv log: name, launches, mean us."""
import csv
import sys
from collections import OrderedDict

for path in sys.argv[1:]:
    rows = [l for l in open(path) if l.startswith('"')]
    agg = OrderedDict()
    for r in csv.DictReader(rows):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("unnamed>::", "")
        v = float(r["Metric Value"].replace(",", "")) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        n, s = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, s + v)
    print(path)
    for k, (n, s) in agg.items():
        print(f"  {k[:70]:70s} {n:4d} x {s / n:10.1f} us")
