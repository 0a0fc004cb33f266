"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes):
per kernel name, launches, mean us, MB read/written per launch.
    python tools/ncu_table.py file.csv [skip_first_n_launches]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr = None
data = collections.OrderedDict()
for r in rows:
    if len(r) > 5 and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        data.setdefault(int(d["ID"]), {"name": d["Kernel Name"].split("(")[0][-40:]})[
            d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
agg = collections.OrderedDict()
for i, m in data.items():
    if i < skip:
        continue
    a = agg.setdefault(m["name"], [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
    a[2] += m.get("dram__bytes_read.sum", 0) / 1e6
    a[3] += m.get("dram__bytes_write.sum", 0) / 1e6
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':42s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'MB rd':>8s} {'MB wr':>8s} {'TB/s':>7s}")
for k, (n, us, rd, wr) in agg.items():
    print(f"{k:42s} {n:4d} {us / n:10.1f} {us / tot:6.1%} {rd / n:8.1f} {wr / n:8.1f} "
          f"{(rd + wr) / us if us else 0:7.2f}")
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
