"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections, csv, sys
agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
    v = float(d["Metric Value"].replace(",", ""))
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(d["Metric Unit"], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(t for _, t in agg.values())
print(f"{'kernel':44s} {'launches':>8s} {'total ms':>10s} {'share':>6s} {'us/launch':>10s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:44]:44s} {n:8d} {t/1e3:10.3f} {100*t/tot:5.1f}% {t/n:10.2f}")
