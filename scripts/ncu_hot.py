"""Summarise an ncu SASS source page (csv): top instructions by stall samples,
with their stall breakdown.   ncu -i X.ncu-rep --page source --csv --print-source sass > s.csv
    python scripts/ncu_hot.py s.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print("total samples", tot)
agg = {c: sum(float(d[c] or 0) for d in data) for c in stall_cols}
print("by reason:", ", ".join(f"{k[6:]}={v / tot:.1%}" for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v))
data.sort(key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))
for d in data[:top]:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    why = sorted(((float(d[c] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{s / tot:6.1%} {d['Address']:>6} {d['Source'][:70]:70s} " + " ".join(f"{n}:{v:.0f}" for v, n in why if v))
