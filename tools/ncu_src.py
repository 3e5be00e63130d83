"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
tot = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
top = sorted(data, key=lambda r: -int(r[idx["Warp Stall Sampling (All Samples)"]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in top:
    n = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    rs = sorted(((int(r[idx[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    print(f"{100*n/tot:5.1f}% {r[idx['Address']]:>6} {r[idx['Source']][:70]:70s} {rs}")
