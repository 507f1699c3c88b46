"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): time share by kernel.
    python scripts/launch_shares.py launches.csv [top]"""
import collections
import csv
import re
import sys

lines = [ln for ln in open(sys.argv[1]) if ln.startswith('"')]  # skip ncu's ==PROF== lines
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
agg = collections.defaultdict(lambda: [0, 0.0, set()])
for r in rows:
    name = re.sub(r"\(CUtensorMap_st.*|\(.*", "", r["Kernel Name"]).replace("dbs::<unnamed>::", "").replace("void ", "").replace("unnamed>::", "")
    v = float(r["Metric Value"]) * (1e3 if r["Metric Unit"] == "us" else 1.0 if r["Metric Unit"] == "ns" else 1e6)
    agg[name][0] += 1
    agg[name][1] += v
    agg[name][2].add(r["Grid Size"])
tot = sum(a[1] for a in agg.values())
print(f"{len(rows)} launches, {tot / 1e3:.1f} us in total (cold-cache, serialised: compare shares)")
print("| share | launches | time (us) | kernel | grids |")
print("|---|---|---|---|---|")
for k, (c, t, g) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"| {100 * t / tot:.1f}% | {c} | {t / 1e3:.1f} | `{k}` | {', '.join(sorted(g))[:40]} |")
