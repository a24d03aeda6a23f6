"""Summarise an ncu source-page CSV (--page source --csv --print-source sass):
stall reasons in total and for the top instructions."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
# the source page may carry a preamble: the header is the first row with "Address"
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
col = {h: i for i, h in enumerate(hdr)}
f = lambda r, h: float(r[col[h]] or 0)
tot = {h: sum(f(r, h) for r in data) for h in reasons}
print("total:", {k[6:]: int(v) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v})
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    top = sorted(((f(r, h), h[6:]) for h in reasons), reverse=True)[:3]
    print(f"{r[col['Address']][-5:]} {int(f(r,'Warp Stall Sampling (All Samples)')):5d} ex={r[col['Instructions Executed']]:>8} "
          f"{r[col['Source']][:60]:60s} " + " ".join(f"{h}={int(v)}" for v, h in top if v))
