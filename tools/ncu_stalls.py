"""Stall-reason totals and the hottest SASS lines of one kernel in an
.ncu-rep (--set full --import-source on).  python tools/ncu_stalls.py rep [top] [kernel_regex]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
kfilter = ["-k", "regex:" + sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
                     + kfilter, capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h) and x[0] != "Address"]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: sum(float(x[h.index(c)] or 0) for x in rows) for c in cols}
alls = sum(tot.values())
print("stall totals (share of samples):")
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {c:24s} {v / alls:6.1%}")
iS = h.index("Warp Stall Sampling (All Samples)")
print("hottest instructions:")
for x in sorted(rows, key=lambda x: -float(x[iS] or 0))[:top]:
    why = max(cols, key=lambda c: float(x[h.index(c)] or 0))
    print(f"  {x[iS]:>6s} {x[0][-5:]} {why[6:]:14s} {x[1][:80]}")
