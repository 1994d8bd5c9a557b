"""Summarise an ncu --page source --print-source sass CSV: top SASS lines by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows[:10]) if "Source" in r)
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
body = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
tot = sum(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in body)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
body.sort(key=lambda r: -float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in body[:n]:
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    top = sorted(((float(r[ix[h]] or 0), h) for h in stalls), reverse=True)[:2]
    print(f"{100*s/tot:5.1f}% {r[ix['Address']]:>6} {r[ix['Source']][:70]:70s} " + " ".join(f"{h[6:]}={v:.0f}" for v, h in top))
