"""Per-CUDA-line stall samples from  ncu --page source --csv --print-source cuda,sass
    python scripts/ncu_lines.py file.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = []
hdr = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr, r))
        try:
            s = float(r[4] or 0)
        except ValueError:
            continue
        st = {h[6:]: float(v or 0) for h, v in zip(hdr, r) if h.startswith("stall_") and "Not Issued" not in h}
        out.append((s, r[0], r[1], st))
tot = sum(o[0] for o in out)
print("total", tot)
for s, ln, src, st in sorted(out, reverse=True)[:top]:
    why = sorted(((v, k) for k, v in st.items()), reverse=True)[:3]
    print(f"{s / tot:6.1%} L{ln:>5} {src.strip()[:80]:80s} " + " ".join(f"{k}:{v:.0f}" for v, k in why if v))
